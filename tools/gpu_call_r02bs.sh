#!/bin/bash
# scrambled work order (2) vs strip-major (0) / run-major (1)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_tb2.py -q -x -p no:cacheprovider -k "work_orders" > gpurun_out/bs_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bs_pytest.log
for i in 1 2; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --order 0,2 >> gpurun_out/bs.jsonl 2>> gpurun_out/bs.err
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --run 120 --order 0,2 >> gpurun_out/bs.jsonl 2>> gpurun_out/bs.err
done
timeout 300 python tools/tb2_probe.py --Lx 4096 --Ly 8192 --steps 40 --preload 1.0 --arith fast --order 1,2 >> gpurun_out/bs.jsonl 2>> gpurun_out/bs.err
timeout 300 python tools/tb2_probe.py --Lx 1024 --Ly 2048 --steps 200 --preload 1.0 --arith fast --order 0,2 >> gpurun_out/bs.jsonl 2>> gpurun_out/bs.err
