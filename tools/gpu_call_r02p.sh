#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/p_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/p_pytest.log
for s in "1920 2048" "1024 2048" "2048 2048" "4096 2048" "4096 8192"; do
  set -- $s
  timeout 300 python tools/tb2_probe.py --Lx $1 --Ly $2 --steps 100 --preload 0.5 --arith fast --run 0,128 >> gpurun_out/p_tb2.jsonl 2>> gpurun_out/p_tb2.err
done
timeout 600 python tools/c1_probe.py --steps 2048 --sizes 256x128 > gpurun_out/p_c1.jsonl 2> gpurun_out/p_c1.err
