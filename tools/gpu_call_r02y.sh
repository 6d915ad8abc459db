#!/bin/bash
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for i in 1 2; do
TLB_LIB_PATH=$PWD/build/norstream/libtlb.so timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 > gpurun_out/y_off$i.json 2> gpurun_out/y_off.err
timeout 300 python tools/tb2_probe.py --steps 200 --preload 1.0 > gpurun_out/y_on$i.json 2> gpurun_out/y_on.err
done
timeout 600 python -m pytest tests/test_gpu_tb2.py tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/y_pytest.log 2>&1
echo "rc=$?" >> gpurun_out/y_pytest.log
