#!/bin/bash
# next-column gather split around level 2 (cfg 9: 19 early, cfg 10: 9 early) vs cfg 1
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --cfg 1,9,10 >> gpurun_out/bg.jsonl 2>> gpurun_out/bg.err
done
timeout 300 python tools/tb2_probe.py --Lx 4096 --Ly 8192 --steps 40 --preload 1.0 --arith fast --cfg 1,9,10 >> gpurun_out/bg.jsonl 2>> gpurun_out/bg.err
