#!/bin/bash
# r02 am: the driver's round-end sequence at HEAD on one B200
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/am_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/am_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/am_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/am_smoke.log
timeout 600 python bench.py --impl reference > gpurun_out/am_ref.json 2> gpurun_out/am_ref.err
timeout 400 python bench.py > gpurun_out/am_bench.json 2> gpurun_out/am_bench.err
