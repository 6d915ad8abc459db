#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 300 python tools/tb2_probe.py --cfg 1 --run 24 --steps 200 --preload 1.0 --arith fast > gpurun_out/g_new.json 2> gpurun_out/g_new.err
TLB_LIB_PATH=$PWD/build/negold/libtlb.so timeout 300 python tools/tb2_probe.py --cfg 1 --run 24 --steps 200 --preload 1.0 --arith fast > gpurun_out/g_negold.json 2> gpurun_out/g_negold.err
