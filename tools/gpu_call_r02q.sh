#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/q_pytest.log
timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/q_pytest2.log 2>&1
echo "rc=$?" >> gpurun_out/q_pytest2.log
