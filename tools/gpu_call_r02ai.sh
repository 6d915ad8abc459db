#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 600 ncu --set full --cache-control none --clock-control none -k regex:"k_site" --launch-skip 4 -c 2 \
  -o gpurun_out/r02ai_c1 -f python tools/small_probe.py --sizes 256x128 --reps 2 > gpurun_out/ai_ncu.log 2>&1
ncu -i gpurun_out/r02ai_c1.ncu-rep --page raw --csv > gpurun_out/r02ai_c1_raw.csv 2>>gpurun_out/ai_ncu.log
