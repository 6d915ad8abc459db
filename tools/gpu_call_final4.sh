# 4 GPUs: multi-GPU parity (NCCL ring 1-D/2-D, peer stores), weak/strong scaling, 1-D vs 2-D tiling
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -p no:cacheprovider 2>&1 | tail -3
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
run() { tag=$1; shift; timeout 300 $R --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 "$@" > gpurun_out/b4_$tag.json 2> gpurun_out/b4_$tag.err; tail -1 gpurun_out/b4_$tag.err | cut -c 1-200; python -c "import json;d=json.loads(open('gpurun_out/b4_$tag.json').read().strip().splitlines()[-1]);print('$tag', d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d.get('other_arith',{}).get('value'), d.get('e2e') and d['e2e'].get('value'), d['clocks'])"; }
run weak_nccl --steps 50 --warmup 5 --cpu-seconds 0
run weak_p2p --steps 50 --warmup 5 --exchange p2p --no-e2e --no-split
run strong_1d --strong --steps 20 --warmup 3 --no-e2e --no-split
run strong_2x2 --strong --steps 20 --warmup 3 --no-e2e --no-split --tiling 2x2
run strong_p2p --strong --steps 20 --warmup 3 --no-e2e --no-split --exchange p2p
