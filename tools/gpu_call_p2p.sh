# 2-GPU: parity of the NCCL ring and the NVLink peer-store step, then both benches
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 tests/dist_run.py 2>&1 | grep -E "tiling=|DIST|Error|error" | head -30
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
for X in nccl p2p; do
timeout 300 $R --master-port 2956$N bench.py --gpus $N --steps 50 --warmup 5 --exchange $X --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bench_${X}_n$N.json 2> gpurun_out/bench_${X}_n$N.err
tail -2 gpurun_out/bench_${X}_n$N.err | cut -c 1-300
python -c "import json;d=json.loads(open('gpurun_out/bench_${X}_n$N.json').read().strip().splitlines()[-1]);print('$X', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d.get('other_arith',{}).get('value'))"
done
