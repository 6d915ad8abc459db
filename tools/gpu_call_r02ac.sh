#!/bin/bash
# r02 ac: ncu --set full of the ring kernels (two in-process ranks on GPU 0) + smoke + bench
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python __graft_entry__.py smoke > gpurun_out/ac_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/ac_smoke.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_peer_step|k_tb2" -c 6 \
  -o gpurun_out/r02ac_peer -f python tools/peer_ncu.py fast on 0 > gpurun_out/ac_ncu_on.log 2>&1
echo "rc=$?" >> gpurun_out/ac_ncu_on.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_peer_step<0, 0>" -c 2 \
  -o gpurun_out/r02ac_peer1 -f python tools/peer_ncu.py fast off 0 > gpurun_out/ac_ncu_off.log 2>&1
echo "rc=$?" >> gpurun_out/ac_ncu_off.log
ncu -i gpurun_out/r02ac_peer.ncu-rep --page raw --csv > gpurun_out/r02ac_ncu_peer_pairs_column_raw.csv 2>>gpurun_out/ac_ncu_on.log
ncu -i gpurun_out/r02ac_peer1.ncu-rep --page raw --csv > gpurun_out/r02ac_ncu_peer_step_column_raw.csv 2>>gpurun_out/ac_ncu_off.log
