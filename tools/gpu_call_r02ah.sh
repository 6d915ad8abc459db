#!/bin/bash
# r02 ah (2 GPUs): full GPU suite (incl. multi-GPU), ncu of the ring kernel at HEAD, smoke
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ah_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ah_pytest.log
CUDA_VISIBLE_DEVICES=0 timeout 300 python __graft_entry__.py smoke > gpurun_out/ah_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ah_smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" -c 3 \
  -o gpurun_out/r02ah_peer -f python tools/peer_ncu.py fast on 0 > gpurun_out/ah_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/ah_ncu.log
ncu -i gpurun_out/r02ah_peer.ncu-rep --page raw --csv > gpurun_out/r02ah_ncu_peer_pairs_column_raw.csv 2>>gpurun_out/ah_ncu.log
