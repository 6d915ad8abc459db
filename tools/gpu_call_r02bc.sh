#!/bin/bash
# run-length cap (512): auto vs fixed runs with the production work order (-1)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for s in "1920 2048" "1024 2048" "4096 2048"; do
  set -- $s
  timeout 300 python tools/tb2_probe.py --Lx $1 --Ly $2 --steps 100 --preload 0.7 --arith fast --order -1 >> gpurun_out/bc.jsonl 2>> gpurun_out/bc.err
done
for s in "4096 8192" "2048 16384" "4096 16384" "8192 16384"; do
  set -- $s
  for run in 0 256 512 1024; do
    timeout 300 python tools/tb2_probe.py --Lx $1 --Ly $2 --steps 20 --preload 0.7 --arith fast --order -1 --run $run >> gpurun_out/bc.jsonl 2>> gpurun_out/bc.err
  done
done
