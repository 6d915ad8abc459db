#!/bin/bash
# r02 b: new parity tests (C2 fast headline vs oracle, C4/C5 macro contract,
# payload golden), tb2 shape sweep, ncu --set full of the step kernels at HEAD,
# bench launch list
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -s \
  -k "c2_headline or face_payload or c5_translation or c4_conservation" > gpurun_out/b_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/b_pytest.log
timeout 600 python tools/tb2_probe.py --cfg 0,1,2,3,4,5,6 --run 64,128,256 --steps 200 > gpurun_out/b_tb2.json 2> gpurun_out/b_tb2.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_site|k_tb2" \
  -o gpurun_out/r02_c2_steps -f python tools/ncu_capture.py > gpurun_out/b_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/b_ncu.log
ncu -i gpurun_out/r02_c2_steps.ncu-rep --page raw --csv > gpurun_out/r02_ncu_c2_column_raw.csv 2>>gpurun_out/b_ncu.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_bench_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-split --no-probe --cpu-seconds 0 --preload 0 > gpurun_out/b_ncu_bench.log 2>&1
