#!/bin/bash
# work order on the strong-scaling tiles (N=4: 2048x16384, N=2: 4096x16384)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for s in "2048 16384" "4096 16384" "4096 8192"; do
  set -- $s
  for o in 0 1 0 1; do
    timeout 300 python tools/tb2_probe.py --Lx $1 --Ly $2 --steps 20 --preload 0.7 --arith fast --order $o >> gpurun_out/bj.jsonl 2>> gpurun_out/bj.err
  done
done
