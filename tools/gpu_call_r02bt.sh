#!/bin/bash
# N=2 default bench line at HEAD (traffic from the SASS-matched ring capture)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29781 bench.py --gpus 2 --steps 100 --warmup 5 > gpurun_out/bt_n2.json 2> gpurun_out/bt_n2.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29782 bench.py --impl reference --gpus 2 --steps 100 --warmup 5 > gpurun_out/bt_n2_ref.json 2> gpurun_out/bt_n2_ref.err
