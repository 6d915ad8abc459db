O=fused_exact_step_neg,fused_fast_step,propagate,fused_exact_step_neg_reload5
python tools/kernel_variants.py --only $O 2>&1 | grep -v "^{"
echo "--- padded"
python tools/kernel_variants.py --only $O --pad 1 2>&1 | grep -v "^{"
echo "--- hints"
TLB_LIB_PATH=paper_1703_00185_b200/libtlb_hints.so python tools/kernel_variants.py --only $O 2>&1 | grep -v "^{"
echo "--- hints padded"
TLB_LIB_PATH=paper_1703_00185_b200/libtlb_hints.so python tools/kernel_variants.py --only $O --pad 1 2>&1 | grep -v "^{"
