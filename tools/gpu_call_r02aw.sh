#!/bin/bash
# r02 aw: HEAD ncu capture of the step kernels (C2) with SASS hashes, bench N=1 +
# launch list, reference arm, C2 work-order A/B (3 rounds)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_site|k_tb2" \
  -o gpurun_out/r02z_c2_steps -f python tools/ncu_capture.py > gpurun_out/aw_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/aw_ncu.log
ncu -i gpurun_out/r02z_c2_steps.ncu-rep --page raw --csv > gpurun_out/r02z_ncu_c2_column_raw.csv 2>>gpurun_out/aw_ncu.log
python tools/ncu_capture.py --hash-only gpurun_out/r02z_ncu_c2_column_raw.csv >> gpurun_out/aw_ncu.log 2>&1
cp gpurun_out/r02z_ncu_c2_column_raw.csv gpurun_out/r02z_ncu_c2_column_raw.csv.sass profiles/ 2>/dev/null
rm -f gpurun_out/r02z_c2_steps.ncu-rep
timeout 400 python bench.py > gpurun_out/aw_bench.json 2> gpurun_out/aw_bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02z_bench_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-split --no-probe --cpu-seconds 0 --preload 0 > gpurun_out/aw_ncu_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/aw_ref.json 2> gpurun_out/aw_ref.err
for i in 1 2 3; do
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --order 0 >> gpurun_out/aw_order.jsonl 2>> gpurun_out/aw.err
  timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 --arith fast --order 1 >> gpurun_out/aw_order.jsonl 2>> gpurun_out/aw.err
done
