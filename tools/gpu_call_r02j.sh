#!/bin/bash
# r02 j (2 GPUs): HEAD ncu of the 1-GPU step kernels (+SASS hashes), bench N=1
# and its launch list, multi-GPU tests, bench N=2 weak, ncu of k_peer_step
# with NVLink bytes (in-process, 2 GPUs)
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/j_topo.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_site|k_tb2" \
  -o gpurun_out/r02j_c2_steps -f python tools/ncu_capture.py > gpurun_out/j_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/j_ncu.log
ncu -i gpurun_out/r02j_c2_steps.ncu-rep --page raw --csv > gpurun_out/r02j_ncu_c2_column_raw.csv 2>>gpurun_out/j_ncu.log
python tools/ncu_capture.py --hash-only gpurun_out/r02j_ncu_c2_column_raw.csv >> gpurun_out/j_ncu.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 400 python bench.py > gpurun_out/j_bench1.json 2> gpurun_out/j_bench1.err
CUDA_VISIBLE_DEVICES=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02j_bench_launches.csv python bench.py --steps 4 --warmup 3 --no-e2e --no-split --no-probe --cpu-seconds 0 --preload 0 > gpurun_out/j_ncu_bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/j_multi.log 2>&1
echo "rc=$?" >> gpurun_out/j_multi.log
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 > gpurun_out/j_bench2.json 2> gpurun_out/j_bench2.err
timeout 600 ncu --set full --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum \
  --clock-control none -k regex:k_peer_step -c 4 -o gpurun_out/r02j_peer -f python tools/peer_ncu.py fast > gpurun_out/j_peer_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/j_peer_ncu.log
ncu -i gpurun_out/r02j_peer.ncu-rep --page raw --csv > gpurun_out/r02j_peer_raw.csv 2>>gpurun_out/j_peer_ncu.log
