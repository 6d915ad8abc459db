#!/bin/bash
# single-step CTA size for small launches (C1 and friends)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python tools/small_probe.py --sizes 256x128,512x256,1024x512 --bs 0,128,64,32 --no-pairs --reps 30 >> gpurun_out/bh.jsonl 2>> gpurun_out/bh.err
done
timeout 600 python tools/c1_probe.py --steps 2048 --sizes 256x128,512x256 >> gpurun_out/bh_c1.jsonl 2>> gpurun_out/bh.err
