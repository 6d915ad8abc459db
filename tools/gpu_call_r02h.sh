#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/tb2_probe.py --cfg 1 --run 32,64,128,240 --order 0,1,2 --steps 200 --preload 0.7 --arith fast > gpurun_out/h_tb2.json 2> gpurun_out/h_tb2.err
timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/h_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/h_pytest.log
