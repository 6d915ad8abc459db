#!/bin/bash
# r02 t (2 GPUs): NVLink + DRAM bytes of the fused peer kernels (single step and pairs)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum
for t in off on; do
  timeout 900 ncu --replay-mode application --clock-control none --metrics $M -k regex:"k_peer_step|k_tb2" -c 12 \
    --csv --log-file gpurun_out/r02t_peer_$t.csv python tools/peer_ncu.py fast $t > gpurun_out/t_$t.log 2>&1
  echo "rc=$?" >> gpurun_out/t_$t.log
done
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 bench.py --gpus 2 --no-e2e --no-split > gpurun_out/t_bench2.json 2> gpurun_out/t_bench2.err
