#!/bin/bash
# edge strips first for periodic Y too: periodic/walls C2 auto + run sweep, tb2 tests
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for per in "--periodic" "" "--periodic"; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast $per >> gpurun_out/ba.jsonl 2>> gpurun_out/ba.err
done
for run in 64 128; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast --periodic --run $run >> gpurun_out/ba.jsonl 2>> gpurun_out/ba.err
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/ba_pytest.log 2>&1
