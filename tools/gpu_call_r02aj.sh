#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python tools/small_probe.py --sizes 256x128,512x256 > gpurun_out/aj_small.jsonl 2> gpurun_out/aj_small.err
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/aj_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/aj_pytest.log
timeout 600 python tools/c1_probe.py --steps 4096 --sizes 256x128 > gpurun_out/aj_c1.jsonl 2> gpurun_out/aj_c1.err
