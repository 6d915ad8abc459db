# 2 GPUs: NVLink halo bandwidth table + planner predictions; strong scaling N=1, N=2
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
timeout 300 $R --master-port 29571 tools/halo_bandwidth.py --out gpurun_out/halo_bw.csv > gpurun_out/halo_bw.json 2> gpurun_out/halo_bw.err
tail -3 gpurun_out/halo_bw.err | cut -c 1-300; cat gpurun_out/halo_bw.csv
timeout 400 python bench.py --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0 > gpurun_out/bench_strong_n1.json 2> gpurun_out/bench_strong_n1.err
tail -2 gpurun_out/bench_strong_n1.err | cut -c 1-300
timeout 300 $R --master-port 29572 bench.py --gpus 2 --strong --steps 20 --warmup 3 --no-e2e --no-split > gpurun_out/bench_strong_n2.json 2> gpurun_out/bench_strong_n2.err
tail -2 gpurun_out/bench_strong_n2.err | cut -c 1-300
for f in bench_strong_n1 bench_strong_n2; do python -c "import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('other_arith',{}).get('value'))"; done
