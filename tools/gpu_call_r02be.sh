#!/bin/bash
# ring two-step kernel (PEER) vs the one-tile kernel: ncu --set full, both ranks on GPU 0
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" -c 4 \
  -o gpurun_out/be_peer -f python tools/peer_ncu.py fast on 0 > gpurun_out/be_ncu.log 2>&1
ncu -i gpurun_out/be_peer.ncu-rep --page raw --csv > gpurun_out/be_peer_raw.csv 2>>gpurun_out/be_ncu.log
ncu -i gpurun_out/be_peer.ncu-rep --page source --csv > gpurun_out/be_peer_source.csv 2>>gpurun_out/be_ncu.log
rm -f gpurun_out/be_peer.ncu-rep
