#!/bin/bash
# pairing threshold: single vs two-step on mid-size tiles (fast)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for s in "512 1024" "768 1024" "1024 1024" "1024 1536" "1536 1024" "2048 512"; do
  set -- $s
  timeout 300 python tools/tb2_probe.py --Lx $1 --Ly $2 --steps 400 --preload 0.7 --arith fast >> gpurun_out/bw.jsonl 2>> gpurun_out/bw.err
done
