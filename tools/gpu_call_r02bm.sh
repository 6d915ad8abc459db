#!/bin/bash
# HEAD check: the driver's round-end sequence (late round 2)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/bm_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/bm_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/bm_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bm_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/bm_smoke.log
timeout 600 python bench.py --impl reference > gpurun_out/bm_ref.json 2> gpurun_out/bm_ref.err
timeout 600 python bench.py > gpurun_out/bm_bench.json 2> gpurun_out/bm_bench.err
