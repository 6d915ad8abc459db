# 4-GPU box: weak and strong scaling lines at N=1,2,4 with the column layout
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
run() { n=$1; tag=$2; shift; shift; timeout 300 $R --nproc-per-node $n --master-port $((29600 + RANDOM % 300)) bench.py --gpus $n "$@" > gpurun_out/s_${tag}.json 2> gpurun_out/s_${tag}.err; python -c "import json;d=json.loads(open('gpurun_out/s_${tag}.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['ms_per_step'], d.get('other_arith',{}).get('value'), d.get('e2e') and d['e2e'].get('value'), d['clocks'])" || tail -3 gpurun_out/s_${tag}.err; }
run 2 weak_n2 --steps 100 --warmup 5 --cpu-seconds 0 --no-split
run 4 weak_n4 --steps 100 --warmup 5 --cpu-seconds 0 --no-split
run 1 strong_n1 --strong --steps 20 --warmup 3 --no-e2e --no-split --cpu-seconds 0
run 2 strong_n2 --strong --steps 20 --warmup 3 --no-e2e --no-split
run 4 strong_n4 --strong --steps 20 --warmup 3 --no-e2e --no-split
