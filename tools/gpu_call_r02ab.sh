#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do timeout 600 python tools/small_probe.py --sizes 256x128,512x256 >> gpurun_out/ab_small.jsonl 2> gpurun_out/ab_small.err; done
