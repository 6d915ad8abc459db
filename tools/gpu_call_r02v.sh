#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/v_pytest.log
(cd build/old && timeout 300 python tools/tb2_probe.py --cfg 1 --run 128 --steps 200 --preload 1.0 --arith fast) > gpurun_out/v_old.json 2> gpurun_out/v_old.err
timeout 300 python tools/tb2_probe.py --cfg 1 --steps 200 --preload 1.0 --arith fast > gpurun_out/v_new.json 2> gpurun_out/v_new.err
