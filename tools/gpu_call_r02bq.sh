#!/bin/bash
# fast pair arithmetic with the odd part folded into the relaxation FMA: rate + parity
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast >> gpurun_out/bq.jsonl 2>> gpurun_out/bq.err
done
timeout 300 python tools/tb2_probe.py --Lx 4096 --Ly 8192 --steps 40 --preload 1.0 --arith fast --order -1 >> gpurun_out/bq.jsonl 2>> gpurun_out/bq.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_tb2.py tests/test_gpu_parity.py -q -x -p no:cacheprovider > gpurun_out/bq_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bq_pytest.log
timeout 600 python tools/drift_probe.py --Lx 1920 --Ly 2048 --checkpoints 100,1000,2000 > gpurun_out/bq_drift.jsonl 2>> gpurun_out/bq.err
