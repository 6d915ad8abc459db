#!/bin/bash
# 4 GPUs after the schedule changes: full GPU suite (multi-GPU included),
# weak (configs[2]) and strong (configs[3]) lines at N = 1, 2, 4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bd_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bd_pytest.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 1 2 4; do
  timeout 400 $R --nproc-per-node $N --master-port $((29700 + N)) bench.py --gpus $N --steps 100 --warmup 5 --cpu-seconds 0 > gpurun_out/bd_weak$N.json 2> gpurun_out/bd_weak$N.err
  timeout 400 $R --nproc-per-node $N --master-port $((29710 + N)) bench.py --gpus $N --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bd_strong$N.json 2> gpurun_out/bd_strong$N.err
done
