#!/bin/bash
# r02 k: multi-step cooperative kernel for small tiles: tests + C1 probe
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multistep.py -x -q -p no:cacheprovider > gpurun_out/k_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/k_pytest.log
timeout 900 python tools/c1_probe.py --steps 2048 > gpurun_out/k_c1.jsonl 2> gpurun_out/k_c1.err
