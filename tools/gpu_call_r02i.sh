#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
(cd build/old && timeout 300 python tools/tb2_probe.py --cfg 1 --run 128 --steps 200 --preload 0.7 --arith fast) > gpurun_out/i_old.json 2> gpurun_out/i_old.err
timeout 300 python tools/tb2_probe.py --cfg 1 --run 64,128 --steps 200 --preload 0.7 --arith fast > gpurun_out/i_new.json 2> gpurun_out/i_new.err
timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/i_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/i_pytest.log
