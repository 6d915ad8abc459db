#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for s in "1920 2048" "4096 8192" "8192 16384"; do
  set -- $s
  timeout 600 python tools/tb2_probe.py --Lx $1 --Ly $2 --steps 40 --preload 1.0 --arith fast --order 0,1,0,1 >> gpurun_out/an_tb2.jsonl 2>> gpurun_out/an.err
done
