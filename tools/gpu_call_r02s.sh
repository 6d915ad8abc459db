#!/bin/bash
# r02 s (4 GPUs): ring pair tests, weak and strong scaling N=2,4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 600 python -m pytest tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/s_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/s_pytest.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -s > gpurun_out/s_multi.log 2>&1
echo "rc=$?" >> gpurun_out/s_multi.log
for n in 2 4; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n > gpurun_out/s_weak$n.json 2> gpurun_out/s_weak$n.err
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --strong --no-e2e --no-split > gpurun_out/s_strong$n.json 2> gpurun_out/s_strong$n.err
done
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --strong --no-e2e --no-split > gpurun_out/s_strong1.json 2> gpurun_out/s_strong1.err
