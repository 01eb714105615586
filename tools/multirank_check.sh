#!/usr/bin/env bash
# Exercises bench.py's N > 1 code paths on a 1-GPU box: (1) one rank with the C ABI's NCCL communicator forced on,
# (2) two ranks sharing the GPU over gloo.  Usage: gpurun -- 'bash tools/multirank_check.sh <out_dir>'
OUT=${1:-gpurun_out/multirank}; mkdir -p "$OUT"
QVK_BENCH_FORCE_COMM=1 timeout 600 python -m torch.distributed.run --nnodes 1 --nproc-per-node 1 \
  --master-addr 127.0.0.1 --master-port 29511 bench.py --config C2 --steps 3 --warmup 2 --no-cpu-baseline \
  > "$OUT/force_comm.log" 2>&1; echo "rc=$?" >> "$OUT/force_comm.log"
QVK_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes 1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29512 bench.py --config C2 --steps 3 --warmup 2 --no-cpu-baseline \
  > "$OUT/share2.log" 2>&1; echo "rc=$?" >> "$OUT/share2.log"
