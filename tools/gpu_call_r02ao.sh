#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_tb2.py tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/ao_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ao_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py --strong --no-e2e --no-split > gpurun_out/ao_strong1.json 2> gpurun_out/ao_strong1.err
for o in 0 1; do
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2970$o bench.py --gpus 2 --strong --no-e2e --no-split --no-compare --tb2-order $o > gpurun_out/ao_strong2_o$o.json 2> gpurun_out/ao_strong2_o$o.err
done
