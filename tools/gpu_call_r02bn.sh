#!/bin/bash
# 4 GPUs: 8-rank rings (in-process on one GPU and over all four), multi-GPU suite
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/bn_local.log 2>&1
echo "rc=$?" >> gpurun_out/bn_local.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/bn_multi.log 2>&1
echo "rc=$?" >> gpurun_out/bn_multi.log
