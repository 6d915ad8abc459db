#!/bin/bash
# r02 f: aligned strip-segment tb2 schedule
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/f_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/f_pytest.log
(cd build/old && timeout 300 python tools/tb2_probe.py --cfg 1 --run 128 --steps 200 --preload 1.0) > gpurun_out/f_old.json 2> gpurun_out/f_old.err
timeout 900 python tools/tb2_probe.py --cfg 0,1,2 --run 24,100000 --steps 200 --preload 1.0 > gpurun_out/f_tb2.json 2> gpurun_out/f_tb2.err
