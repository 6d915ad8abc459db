#!/bin/bash
# 4 GPUs after the run-major threshold change: full GPU suite, strong N = 1, 2, 4, C5 bench split
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bk_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bk_pytest.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 1 2 4; do
  timeout 400 $R --nproc-per-node $N --master-port $((29750 + N)) bench.py --gpus $N --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bk_strong$N.json 2> gpurun_out/bk_strong$N.err
done
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/tb2_probe.py --Lx 4096 --Ly 8192 --steps 40 --preload 1.0 --arith fast,exact --order -1 > gpurun_out/bk_c5.jsonl 2>> gpurun_out/bk.err
