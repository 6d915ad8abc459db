#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/ae_local.log 2>&1
echo "rc=$?" >> gpurun_out/ae_local.log
for i in 1 2; do
(cd build/prev && timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2957$i bench.py --gpus 2 --no-e2e --no-split --no-compare) > gpurun_out/ae_prev$i.json 2> gpurun_out/ae_prev.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2958$i bench.py --gpus 2 --no-e2e --no-split --no-compare > gpurun_out/ae_new$i.json 2> gpurun_out/ae_new.err
done
