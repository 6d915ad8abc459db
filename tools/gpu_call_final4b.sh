# final 4-GPU check: full GPU suite (multi-GPU tests included), N=2 and N=4 default benches
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for N in 2 4; do
timeout 300 $R --nproc-per-node $N --master-port $((29650 + N)) bench.py --gpus $N --steps 100 --warmup 5 --cpu-seconds 0 > gpurun_out/final_n$N.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/final_n$N.json').read());print('N=$N', d['value'], d['config']['exchange'], d['e2e']['value'], d['gpu_launches'], d['clocks']['sm_mhz'])"
done
