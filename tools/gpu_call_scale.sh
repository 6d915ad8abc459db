# N-GPU scaling: weak (configs[2]) and strong (configs[3]) benches under torchrun
N=${1:-4}
R="python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1"
timeout 300 $R --master-port 29541 bench.py --gpus $N --steps 50 --warmup 5 > gpurun_out/bench_weak_n$N.json 2> gpurun_out/bench_weak_n$N.err
tail -3 gpurun_out/bench_weak_n$N.err | cut -c 1-300
timeout 300 $R --master-port 29542 bench.py --gpus $N --steps 20 --warmup 3 --strong --no-e2e --no-split > gpurun_out/bench_strong_n$N.json 2> gpurun_out/bench_strong_n$N.err
tail -3 gpurun_out/bench_strong_n$N.err | cut -c 1-300
cat gpurun_out/bench_weak_n$N.json gpurun_out/bench_strong_n$N.json | cut -c 1-700
