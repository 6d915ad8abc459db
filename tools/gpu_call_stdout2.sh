# N=2: the bench's stdout must be exactly one JSON line per arm
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29611 bench.py --gpus 2 --steps 50 --warmup 5 --cpu-seconds 0 > gpurun_out/o2.json 2> gpurun_out/o2.err
timeout 300 $R --master-port 29612 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/r2.json 2> gpurun_out/r2.err
for f in gpurun_out/o2.json gpurun_out/r2.json; do echo "$f: $(wc -l < $f) line(s)"; python -c "import json; [json.loads(l) for l in open('$f')]; print('parses')"; done
python -c "import json; d=json.loads(open('gpurun_out/o2.json').read()); print(d['value'], d['gpu_launches'], d['clocks'], d['e2e']['value'])"
