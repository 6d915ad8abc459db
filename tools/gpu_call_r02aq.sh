#!/bin/bash
# split two-step kernel (cfg 7): parity and rate against cfg 1
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_tb2.py -x -q -p no:cacheprovider -k "split or every_shape" > gpurun_out/aq_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/aq_pytest.log
timeout 600 python tools/tb2_probe.py --steps 200 --preload 1.5 --arith fast --cfg 1,7,1,7 > gpurun_out/aq_tb2.jsonl 2> gpurun_out/aq.err
