#!/bin/bash
# column-layout specialised two-step kernel (cfg 1, COL) vs generic (soa layout
# forces the generic kernel): A/B in one process
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/av_pytest.log 2>&1
timeout 600 python tools/tb2_probe.py --steps 200 --preload 1.5 --arith fast --cfg 1 --col 1,0,1,0 > gpurun_out/av_tb2.jsonl 2> gpurun_out/av.err
