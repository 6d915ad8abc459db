#!/bin/bash
# 4 GPUs: short border runs for the ring kernel -- peer/tb2 tests, multi-GPU tests, strong and weak lines
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_peer_local.py tests/test_gpu_tb2.py -x -q -p no:cacheprovider > gpurun_out/bl_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bl_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/bl_multi.log 2>&1
echo "rc=$?" >> gpurun_out/bl_multi.log
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
  timeout 400 $R --nproc-per-node $N --master-port $((29760 + N)) bench.py --gpus $N --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bl_strong$N.json 2> gpurun_out/bl_strong$N.err
  timeout 400 $R --nproc-per-node $N --master-port $((29770 + N)) bench.py --gpus $N --steps 100 --warmup 5 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bl_weak$N.json 2> gpurun_out/bl_weak$N.err
done
