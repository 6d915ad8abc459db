# strong scaling 8192x16384 at N=1/2/4 with the final code (default exchange)
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 1 2 4; do
timeout 300 $R --nproc-per-node $N --master-port $((29660 + N)) bench.py --gpus $N --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/strong_final_n$N.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/strong_final_n$N.json').read());print('N=$N', d['value'], d['ms_per_step'], d['config']['exchange'], d['clocks']['sm_mhz'])"
done
