#!/bin/bash
# periodic-Y two-step slowdown: init dependence + ncu (walls vs periodic, run 128)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for init in uniform random; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast --periodic --run 128 --init $init >> gpurun_out/az_per.jsonl 2>> gpurun_out/az.err
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 0.7 --arith fast --run 128 --init $init >> gpurun_out/az_per.jsonl 2>> gpurun_out/az.err
done
for per in "" "--periodic"; do
  tag=w; [ -n "$per" ] && tag=p
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_tb2" \
    -o gpurun_out/az_$tag -f python tools/ncu_capture.py --what pair --arith fast --run 128 $per > gpurun_out/az_ncu_$tag.log 2>&1
  ncu -i gpurun_out/az_$tag.ncu-rep --page raw --csv > gpurun_out/az_${tag}_raw.csv 2>>gpurun_out/az_ncu_$tag.log
  ncu -i gpurun_out/az_$tag.ncu-rep --page source --csv > gpurun_out/az_${tag}_source.csv 2>>gpurun_out/az_ncu_$tag.log
  rm -f gpurun_out/az_$tag.ncu-rep
done
