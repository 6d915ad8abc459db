# configs[4] (C5, 4096x8192): fused vs split kernels, event timing + ncu counters
timeout 600 python -m pytest tests/test_gpu_acceptance.py -q -p no:cacheprovider 2>&1 | tail -2
V="python tools/kernel_variants.py --Lx 4096 --Ly 8192 --reps 5 --only propagate,collide_exact_inplace,collide_fast_inplace,fused_exact_step_neg,fused_fast_step"
timeout 600 $V > gpurun_out/c5_variants.log 2>&1; cat gpurun_out/c5_variants.log | grep -v "^{"
P="python tools/kernel_variants.py --Lx 4096 --Ly 8192 --reps 1 --only propagate,collide_exact_inplace,collide_fast_inplace,fused_exact_step_neg,fused_fast_step"
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second"
timeout 600 ncu --metrics $M --clock-control none -k regex:k_site --csv --log-file gpurun_out/c5_ncu.csv $P > gpurun_out/c5_ncu.log 2>&1
tail -2 gpurun_out/c5_ncu.log
