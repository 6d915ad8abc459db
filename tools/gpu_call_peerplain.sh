# peer step with the branch-free gather in the bands: parity (N=4 torchrun) + strong/weak A/B
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29552 tests/dist_run.py 2>&1 | grep -E "ok=False|DIST|Error|Traceback" | head
bash tools/gpu_call_ab_strong.sh 4 2
bash tools/gpu_call_ab.sh 4 2
