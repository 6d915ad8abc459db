#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/ad_local.log 2>&1
echo "rc=$?" >> gpurun_out/ad_local.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -s > gpurun_out/ad_multi.log 2>&1
echo "rc=$?" >> gpurun_out/ad_multi.log
