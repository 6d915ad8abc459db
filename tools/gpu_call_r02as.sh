#!/bin/bash
# split two-step kernel (cfg 7) after predicated stores: rate vs cfg 1 + source page
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 python tools/tb2_probe.py --steps 200 --preload 1.5 --arith fast --cfg 1,7 > gpurun_out/as_tb2.jsonl 2> gpurun_out/as.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" \
  -o gpurun_out/as_split python tools/ncu_capture.py --what pair --arith fast --cfg 7 > gpurun_out/as_ncu.log 2>&1
ncu -i gpurun_out/as_split.ncu-rep --page source --csv > gpurun_out/as_split_source.csv 2>>gpurun_out/as_ncu.log
ncu -i gpurun_out/as_split.ncu-rep > gpurun_out/as_split_details.txt 2>>gpurun_out/as_ncu.log
rm -f gpurun_out/as_split.ncu-rep
