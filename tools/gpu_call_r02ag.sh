#!/bin/bash
# r02 ag: ncu counters for the north-star split targets on C5 (4096x8192): propagate HBM, collide FP64
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:"k_site" -c 4 -o gpurun_out/r02ag_c5 -f \
  python tools/kernel_variants.py --Lx 4096 --Ly 8192 --reps 1 --only propagate,collide_exact_inplace,collide_fast_inplace,fused_exact_step_neg > gpurun_out/ag_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/ag_ncu.log
ncu -i gpurun_out/r02ag_c5.ncu-rep --page raw --csv > gpurun_out/r02ag_ncu_c5_split_raw.csv 2>>gpurun_out/ag_ncu.log
