"""torchrun worker for the stalled-neighbour test (2 processes).

    tests/dist_stall.py nccl|p2p

Both ranks step together, then rank 1 stops stepping while rank 0 queues two
more steps: rank 0's exchange can never complete.
  nccl: rank 0's synchronize() gives up after the fabric timeout, aborts the
        NCCL ring (releasing the stalled NCCL kernels) and raises
        DeadlockError naming rank 0;
  p2p:  the step kernel's border blocks give up after their bounded wait
        (the fabric timeout, tlb_peer_set_timeout) and flag PEER_TIMEOUT;
        collect() raises DeadlockError naming rank 0.
The one-process-per-GPU analog of the reference's deadlock detection
(runtime.py:146-149, tests/test_runtime.py).  Prints "STALL OK".
"""
import os
import sys
import time

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    assert world == 2
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    tile = tl.decompose(96, 40, world, "1d")[rank]
    mode = sys.argv[1] if len(sys.argv) > 1 else "nccl"
    fabric = tl.DistFabric(timeout=4.0)
    w = tl.RankWorker(tile, vs, p, fabric, device=dev, schedule="overlapped", exchange=mode)
    assert w.exchange_mode == mode
    w.load_block(torch.full((vs.Q, tile.Lx, tile.Ly), 1.0 / vs.Q, dtype=torch.float64,
                            device=dev) * torch.as_tensor(vs.w * vs.Q, device=dev)[:, None, None])
    for s in range(2):
        for phase in ("step_begin", "step_mid", "step_end"):
            getattr(w, phase)(s)
    w.synchronize()
    ok = True
    if rank == 0:
        for s in range(2, 2 + (2 if mode == "nccl" else 6)):   # p2p: later steps fail fast
            for phase in ("step_begin", "step_mid", "step_end"):
                getattr(w, phase)(s)
        t0 = time.monotonic()
        try:
            w.synchronize()
            w.collect()
            ok = False
            print("rank 0: stalled step completed?!", flush=True)
        except tl.DeadlockError as exc:
            waited = time.monotonic() - t0
            # p2p: one 4 s bounded wait, then the sticky flag fails the
            # other queued steps at once (5 waits would take 20 s)
            ok = exc.rank == 0 and 3.5 < waited < (30.0 if mode == "nccl" else 12.0)
            print(f"rank 0 ({mode}): DeadlockError after {waited:.1f} s: {exc}", flush=True)
    flag = torch.tensor([int(ok)], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)     # torch's own communicator
    fabric.abort_ring()                             # local, never waits on the peer
    dist.destroy_process_group()
    if rank == 0 and flag.item() == 1:
        print("STALL OK", flush=True)
    sys.exit(0 if flag.item() == 1 else 1)


if __name__ == "__main__":
    main()
