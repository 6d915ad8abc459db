# 4 GPUs: 2-D peer-store parity (torchrun dist_run, incl. (1,4) and (2,2) p2p), then 2x2 benches
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 tests/dist_run.py 2>&1 | grep -E "tiling=|DIST|Error|error|Traceback" | head -30
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
i=0
for X in nccl p2p nccl p2p; do
i=$((i+1))
timeout 300 $R --master-port $((29580 + i)) bench.py --gpus 4 --strong --tiling 2x2 --steps 40 --warmup 3 --exchange $X --no-e2e --no-split --cpu-seconds 0 --no-compare > gpurun_out/b2d_${X}_$i.json 2> gpurun_out/b2d_${X}_$i.err
python -c "import json;d=json.loads(open('gpurun_out/b2d_${X}_$i.json').read());print('2x2 strong', '$X', d['value'], d['ms_per_step'], d['config']['exchange'], d['gpu_launches'])" || tail -3 gpurun_out/b2d_${X}_$i.err
done
