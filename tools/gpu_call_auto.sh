# exchange="auto" choices: weak (short tiles -> peer stores) and strong (tall tiles -> ring)
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for args in "--steps 100" "--strong --steps 20"; do
timeout 300 $R --nproc-per-node 4 --master-port $((29720 + RANDOM % 50)) bench.py --gpus 4 $args --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/auto.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/auto.json').read());print('$args', d['value'], d['ms_per_step'], d['config']['exchange'])"
done
