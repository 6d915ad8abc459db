# N GPUs: alternate NCCL ring / peer-store benches R times (weak 1920x2048 per GPU)
N=${1:-2}; REPS=${2:-3}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
for k in $(seq $REPS); do for X in nccl p2p; do
i=$((i+1))
timeout 300 $R --master-port $((29600 + i)) bench.py --gpus $N --steps 200 --warmup 5 --exchange $X --no-e2e --no-split --cpu-seconds 0 --no-compare > gpurun_out/ab_${X}_$i.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/ab_${X}_$i.json').read());print('$X', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['clocks'].get('power_w_median'))"
done; done
