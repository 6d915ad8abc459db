#!/bin/bash
# ring two-step kernel with one (coherent) load path: ncu duration on GPU 0, peer tests, N=2 weak bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_tb2<" -c 2 \
  -o gpurun_out/bf_peer -f python tools/peer_ncu.py fast on 0 > gpurun_out/bf_ncu.log 2>&1
ncu -i gpurun_out/bf_peer.ncu-rep --page raw --csv > gpurun_out/bf_peer_raw.csv 2>>gpurun_out/bf_ncu.log
rm -f gpurun_out/bf_peer.ncu-rep
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/bf_pytest.log 2>&1
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 400 $R --nproc-per-node 2 --master-port 29722 bench.py --gpus 2 --steps 100 --warmup 5 --cpu-seconds 0 --no-e2e --no-split > gpurun_out/bf_weak2.json 2> gpurun_out/bf_weak2.err
timeout 400 $R --nproc-per-node 2 --master-port 29723 bench.py --gpus 2 --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bf_strong2.json 2> gpurun_out/bf_strong2.err
