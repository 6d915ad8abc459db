#!/bin/bash
# source-level ncu of the headline two-step kernel (cfg 1, fast) for the instruction mix
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" \
  -o gpurun_out/at_c1 python tools/ncu_capture.py --what pair --arith fast --cfg 1 > gpurun_out/at_ncu.log 2>&1
ncu -i gpurun_out/at_c1.ncu-rep --page source --csv > gpurun_out/at_c1_source.csv 2>>gpurun_out/at_ncu.log
ncu -i gpurun_out/at_c1.ncu-rep --page source --csv --print-source cuda > gpurun_out/at_c1_cuda.csv 2>>gpurun_out/at_ncu.log
ncu -i gpurun_out/at_c1.ncu-rep > gpurun_out/at_c1_details.txt 2>>gpurun_out/at_ncu.log
ncu -i gpurun_out/at_c1.ncu-rep --page raw --csv > gpurun_out/at_c1_raw.csv 2>>gpurun_out/at_ncu.log
rm -f gpurun_out/at_c1.ncu-rep
