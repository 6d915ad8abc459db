#!/bin/bash
# r02 d: static cost-balanced tb2 schedule + OR-based negatives test
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tb2.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/d_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/d_pytest.log
timeout 900 python tools/tb2_probe.py --cfg 0,1,2 --run 8,24,64 --steps 200 --preload 1.0 > gpurun_out/d_tb2.json 2> gpurun_out/d_tb2.err
timeout 400 python bench.py --no-e2e --cpu-seconds 0 > gpurun_out/d_bench.json 2> gpurun_out/d_bench.err
