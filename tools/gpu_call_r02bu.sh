#!/bin/bash
# cluster-pair two-step kernel (cfg 9): parity, then rate vs cfg 1
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_tb2.py -q -x -p no:cacheprovider -k "every_shape" > gpurun_out/bu_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bu_pytest.log
for i in 1 2; do
timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast,exact --cfg 1,9 >> gpurun_out/bu.jsonl 2>> gpurun_out/bu.err
done
timeout 300 python tools/tb2_probe.py --Lx 4096 --Ly 8192 --steps 40 --preload 1.0 --arith fast --cfg 1,9 --order -1 >> gpurun_out/bu.jsonl 2>> gpurun_out/bu.err
