# N GPUs strong 8192x16384: alternate NCCL ring / peer stores R times
N=${1:-4}; REPS=${2:-2}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
i=0
for k in $(seq $REPS); do for X in nccl p2p; do
i=$((i+1))
timeout 300 $R --master-port $((29700 + i)) bench.py --gpus $N --strong --steps 30 --warmup 3 --exchange $X --no-e2e --no-split --cpu-seconds 0 --no-compare > gpurun_out/abs_${X}_$i.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/abs_${X}_$i.json').read());print('$X', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'])"
done; done
