#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -s -k "bench_config or nccl_ring_bitwise" > gpurun_out/al_multi.log 2>&1
echo "rc=$?" >> gpurun_out/al_multi.log
