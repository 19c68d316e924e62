mkdir -p gpurun_out
for args in "--workload qft" "--workload qft --fusion tolerance" "--workload random --fusion tolerance" "--workload controlled --fusion passes"; do
  timeout 600 python bench.py $args --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-secondary > gpurun_out/b.json 2> gpurun_out/b.err; echo "$args rc=$?"
  python - <<'PY'
import json
d=json.load(open('gpurun_out/b.json'))
print(d['config']['workload'][:40], d['config']['fusion'], d['ms_per_step'], d['value'], d['roofline']['kernel'][:40], d['roofline']['frac'], d['self_check']['ok'])
PY
done
python -m paper_1601_07195_b200 qft-bench --help > /dev/null 2>&1; echo cli rc=$?
