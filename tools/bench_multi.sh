#!/bin/bash
# Multi-GPU measurement matrix for one 8xB200 node (not runnable on the one-GPU gpurun boxes).
#   bash tools/bench_multi.sh [out_dir]
# Weak scaling of the default sweep (N = 1, 2, 4, 8; n = 30 + log2 N), BASELINE config 4
# (random, 3 global qubits at N = 8; strong scaling at n = 32) with in-place exchanges, with
# global<->local swaps (--remap) and over the NCCL send/recv data plane, and config 5 (QFT,
# passes; unfused with and without the diagonal fast path).
O=${1:-gpurun_out/multi}
mkdir -p $O
run() {  # run <name> <nproc> <bench args...>
  local name=$1 np=$2; shift 2
  if [ "$np" = 1 ]; then
    python bench.py "$@" --out $O/$name.json > $O/$name.log 2>&1
  else
    python -m torch.distributed.run --nnodes=1 --nproc-per-node $np --master-addr 127.0.0.1 \
      --master-port $((29500 + RANDOM % 1000)) bench.py --gpus $np "$@" --out $O/$name.json > $O/$name.log 2>&1
  fi
}
for N in 1 2 4 8; do run sweep_$N $N; done
for N in 1 2 4 8; do run random32_$N $N --workload random --qubits 32 --fusion passes --no-e2e; done
run random36 8 --workload random --qubits 36 --fusion passes --no-e2e
run random36_remap 8 --workload random --qubits 36 --fusion passes --no-e2e --remap
run random36_nccl 8 --workload random --qubits 36 --fusion passes --no-e2e --data-plane nccl
run qft34_passes 8 --workload qft --qubits 34 --no-e2e
run qft34_unfused 8 --workload qft --qubits 34 --fusion none --no-e2e --steps 2
run qft34_unfused_diag 8 --workload qft --qubits 34 --fusion none --no-e2e --steps 2 --diagonal-local
echo done
