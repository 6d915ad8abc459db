# C5 (4096x8192) with the column layout: events + ncu counters; C2 layout study incl. AoS
bash tools/gpu_call_c5.sh
for L in aos soa column; do echo "--- C2 $L"; python tools/kernel_variants.py --reps 20 --layout $L --only propagate,fused_exact_step_neg,fused_fast_step | grep -v "^{"; done
