set -x
O=gpurun_out/benchall
mkdir -p $O
python bench.py --out $O/sweep.json > $O/sweep.log 2>&1
python bench.py --workload controlled --out $O/controlled.json > $O/controlled.log 2>&1
python bench.py --workload random --out $O/random.json > $O/random.log 2>&1
python bench.py --workload random --fusion passes --out $O/random_passes.json > $O/random_passes.log 2>&1
python bench.py --workload controlled --fusion passes --out $O/controlled_passes.json > $O/controlled_passes.log 2>&1
python bench.py --workload qft --out $O/qft.json > $O/qft.log 2>&1
python bench.py --impl reference --out $O/reference.json > $O/reference.log 2>&1
echo done
