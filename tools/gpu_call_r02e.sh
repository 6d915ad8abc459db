#!/bin/bash
# r02 e: A/B old (dynamic schedule) vs new tb2 on the same box + ncu of new tb2 fast
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
(cd build/old && timeout 300 python tools/tb2_probe.py --cfg 1 --run 128 --steps 200 --preload 1.0 --arith fast) > gpurun_out/e_old.json 2> gpurun_out/e_old.err
timeout 300 python tools/tb2_probe.py --cfg 1 --run 24 --steps 200 --preload 1.0 --arith fast > gpurun_out/e_new.json 2> gpurun_out/e_new.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" \
  -o gpurun_out/r02e_tb2 -f python tools/ncu_capture.py --what pair --arith fast > gpurun_out/e_ncu.log 2>&1
ncu -i gpurun_out/r02e_tb2.ncu-rep --page raw --csv > gpurun_out/r02e_tb2_raw.csv 2>>gpurun_out/e_ncu.log
