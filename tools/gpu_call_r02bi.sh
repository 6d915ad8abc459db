#!/bin/bash
# 4 GPUs, HEAD: full GPU suite, ring-kernel ncu capture with SASS sidecar,
# weak (configs[2]) and strong (configs[3]) lines at N = 1, 2, 4
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/bi_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bi_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" -c 4 \
  -o gpurun_out/bi_peer -f python tools/peer_ncu.py fast on 0 > gpurun_out/bi_ncu.log 2>&1
ncu -i gpurun_out/bi_peer.ncu-rep --page raw --csv > gpurun_out/r02zb_ncu_peer_pairs_column_raw.csv 2>>gpurun_out/bi_ncu.log
python tools/ncu_capture.py --hash-only gpurun_out/r02zb_ncu_peer_pairs_column_raw.csv >> gpurun_out/bi_ncu.log 2>&1
rm -f gpurun_out/bi_peer.ncu-rep
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 1 2 4; do
  timeout 400 $R --nproc-per-node $N --master-port $((29730 + N)) bench.py --gpus $N --steps 100 --warmup 5 --cpu-seconds 0 > gpurun_out/bi_weak$N.json 2> gpurun_out/bi_weak$N.err
  timeout 400 $R --nproc-per-node $N --master-port $((29740 + N)) bench.py --gpus $N --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bi_strong$N.json 2> gpurun_out/bi_strong$N.err
done
