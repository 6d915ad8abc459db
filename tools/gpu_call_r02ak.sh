#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 > gpurun_out/ak_base$i.json 2> gpurun_out/ak.err
TLB_LIB_PATH=$PWD/build/aeo/libtlb.so timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 > gpurun_out/ak_aeo$i.json 2>> gpurun_out/ak.err
done
