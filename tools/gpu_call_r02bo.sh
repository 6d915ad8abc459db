#!/bin/bash
# long-run drift of fast (two-step) vs exact (bitwise) arithmetic
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python tools/drift_probe.py --Lx 1920 --Ly 2048 --checkpoints 20,100,500,1000,2000 > gpurun_out/bo_c2.jsonl 2> gpurun_out/bo.err
timeout 900 python tools/drift_probe.py --Lx 256 --Ly 128 --checkpoints 100,1000,5000,10000 > gpurun_out/bo_c1.jsonl 2>> gpurun_out/bo.err
