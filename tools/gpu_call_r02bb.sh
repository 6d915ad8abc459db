#!/bin/bash
# two-step run length across the configs' tile shapes (walls, fast)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for s in "1024 2048" "4096 2048" "4096 8192" "2048 16384" "4096 16384" "8192 16384"; do
  set -- $s
  for run in 0 128 256 512 1024; do
    [ "$run" -ge "$1" ] && continue
    timeout 300 python tools/tb2_probe.py --Lx $1 --Ly $2 --steps 20 --preload 0.7 --arith fast --run $run >> gpurun_out/bb.jsonl 2>> gpurun_out/bb.err
  done
done
