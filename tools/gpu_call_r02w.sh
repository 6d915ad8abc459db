#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" -c 1 \
  -o gpurun_out/r02w_tb2 -f python tools/ncu_capture.py --what pair --arith fast > gpurun_out/w_ncu.log 2>&1
ncu -i gpurun_out/r02w_tb2.ncu-rep --page source --csv --print-source sass > gpurun_out/r02w_tb2_src.csv 2>>gpurun_out/w_ncu.log
ncu -i gpurun_out/r02w_tb2.ncu-rep --page source --csv --print-source cuda > gpurun_out/r02w_tb2_cuda.csv 2>>gpurun_out/w_ncu.log
ncu -i gpurun_out/r02w_tb2.ncu-rep --page raw --csv > gpurun_out/r02w_tb2_raw.csv 2>>gpurun_out/w_ncu.log
