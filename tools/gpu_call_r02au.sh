#!/bin/bash
# split two-step kernels: with (cfg 7) and without (cfg 8) the register prefetch, vs cfg 1
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python tools/tb2_probe.py --steps 200 --preload 1.5 --arith fast --cfg 1,7,8 > gpurun_out/au_tb2.jsonl 2> gpurun_out/au.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider -k "split or every_shape" > gpurun_out/au_pytest.log 2>&1
