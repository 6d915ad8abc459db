#!/bin/bash
# two-step run length: periodic-Y C2 sweep, C5 walls sweep
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for run in 64 96 120 128 160 240; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast --periodic --run $run >> gpurun_out/ay_per.jsonl 2>> gpurun_out/ay.err
done
for run in 0 128 256 512 1024; do
  timeout 300 python tools/tb2_probe.py --Lx 4096 --Ly 8192 --steps 40 --preload 0.7 --arith fast --run $run >> gpurun_out/ay_c5.jsonl 2>> gpurun_out/ay.err
done
