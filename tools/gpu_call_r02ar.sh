#!/bin/bash
# split two-step kernel (cfg 7): rate vs cfg 1, ncu --set full of one launch
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python tools/tb2_probe.py --steps 200 --preload 1.5 --arith fast --cfg 1,7 > gpurun_out/ar_tb2.jsonl 2> gpurun_out/ar.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" \
  -o gpurun_out/ar_split python tools/ncu_capture.py --what pair --arith fast --cfg 7 > gpurun_out/ar_ncu.log 2>&1
ncu -i gpurun_out/ar_split.ncu-rep --page raw --csv > gpurun_out/ar_split_raw.csv 2>>gpurun_out/ar_ncu.log
ncu -i gpurun_out/ar_split.ncu-rep --page source --csv > gpurun_out/ar_split_source.csv 2>>gpurun_out/ar_ncu.log
ncu -i gpurun_out/ar_split.ncu-rep > gpurun_out/ar_split_details.txt 2>>gpurun_out/ar_ncu.log
