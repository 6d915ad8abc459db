# 1-GPU: GPU suite with the column layout default, layout A/B, bench, launch list, ncu of the step kernels
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
for L in soa column; do echo "--- $L"; python tools/kernel_variants.py --reps 30 --layout $L --only fused_exact_step_neg,fused_fast_step,propagate,collide_fast_inplace | grep -v "^{"; done
timeout 300 python bench.py > gpurun_out/bench43.json 2> gpurun_out/bench43.err; tail -2 gpurun_out/bench43.err
B="python bench.py --steps 20 --warmup 3 --cpu-seconds 0 --no-e2e --no-split --no-compare --no-probe --preload 0"
timeout 300 $B > gpurun_out/b_small.log 2>&1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches43.csv $B > gpurun_out/ncu_launch.log 2>&1
P="python tools/prof_fused.py --layout column --only fused_exact_step_neg,fused_fast_step"
timeout 300 $P > gpurun_out/p_small.log 2>&1 && timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_site -s 1 -c 3 -o gpurun_out/prof_step_column $P > gpurun_out/ncu2.log 2>&1
tail -2 gpurun_out/ncu2.log
