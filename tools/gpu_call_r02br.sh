#!/bin/bash
# C2 wall-strip run length: (light run, wall run) = (128, 64) default vs (120, 80 / 96 / 64)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --run 0 --run-h 0 >> gpurun_out/br.jsonl 2>> gpurun_out/br.err
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --run 120 --run-h 80,96,72 >> gpurun_out/br.jsonl 2>> gpurun_out/br.err
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --run 128 --run-h 96,128 >> gpurun_out/br.jsonl 2>> gpurun_out/br.err
done
