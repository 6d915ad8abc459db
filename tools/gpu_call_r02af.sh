#!/bin/bash
# r02 af (4 GPUs): final scaling lines at HEAD (weak + strong, N=1,2,4)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --no-e2e --no-split > gpurun_out/af_weak1.json 2> gpurun_out/af_weak1.err
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --strong --no-e2e --no-split > gpurun_out/af_strong1.json 2> gpurun_out/af_strong1.err
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2960$n bench.py --gpus $n > gpurun_out/af_weak$n.json 2> gpurun_out/af_weak$n.err
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2961$n bench.py --gpus $n --strong --no-e2e --no-split > gpurun_out/af_strong$n.json 2> gpurun_out/af_strong$n.err
done
