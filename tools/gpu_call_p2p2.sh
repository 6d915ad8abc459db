# N GPUs: parity of the NCCL ring and the NVLink peer-store step, then both benches alternated
N=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29551 tests/dist_run.py 2>&1 | grep -E "tiling=|DIST|Error|error" | head -30
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
for X in nccl p2p nccl p2p; do
i=$((i+1))
timeout 300 $R --master-port $((29570 + i)) bench.py --gpus $N --steps 200 --warmup 5 --exchange $X --no-e2e --no-split --cpu-seconds 0 --no-compare > gpurun_out/bench_${X}_n${N}_$i.json 2> gpurun_out/bench_${X}_n${N}_$i.err
python -c "import json;d=json.loads(open('gpurun_out/bench_${X}_n${N}_$i.json').read().strip().splitlines()[-1]);print('$X', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/bench_${X}_n${N}_$i.err
done
