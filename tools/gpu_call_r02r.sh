#!/bin/bash
# r02 r (2 GPUs): multi-GPU tests incl. ring pairs over IPC, bench N=2 weak (pairs), N=2 nccl
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider -s > gpurun_out/r_multi.log 2>&1
echo "rc=$?" >> gpurun_out/r_multi.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 2 > gpurun_out/r_bench2.json 2> gpurun_out/r_bench2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29522 bench.py --gpus 2 --strong --no-e2e --no-split > gpurun_out/r_bench2s.json 2> gpurun_out/r_bench2s.err
