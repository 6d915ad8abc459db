#!/bin/bash
# HEAD check from a fresh container: the driver's round-end sequence
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/ap_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/ap_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/ap_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ap_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/ap_smoke.log
timeout 600 python bench.py --impl reference > gpurun_out/ap_ref.json 2> gpurun_out/ap_ref.err
timeout 600 python bench.py > gpurun_out/ap_bench.json 2> gpurun_out/ap_bench.err
