#!/bin/bash
# r02 c: tb2 occupancy variants (no register prefetch, more warps)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/tb2_probe.py --cfg 1,7,8,9,10,11 --run 64,128,256 --steps 200 --preload 1.0 > gpurun_out/c_tb2.json 2> gpurun_out/c_tb2.err
timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/c_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/c_pytest.log
