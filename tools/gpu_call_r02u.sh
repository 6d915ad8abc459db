#!/bin/bash
# r02 u (2 GPUs): multi-GPU tests (in-process pairs on 2 GPUs), peer-local, NVLink bytes
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_peer_local.py -x -q -p no:cacheprovider > gpurun_out/u_tests.log 2>&1
echo "rc=$?" >> gpurun_out/u_tests.log
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
for t in off on; do
  timeout 900 ncu --replay-mode application --clock-control none --metrics $M -k regex:"k_peer_step|k_tb2" -c 12 \
    --csv --log-file gpurun_out/r02u_peer_$t.csv python tools/peer_ncu.py fast $t > gpurun_out/u_$t.log 2>&1
  echo "rc=$?" >> gpurun_out/u_$t.log
done
