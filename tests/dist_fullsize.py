"""torchrun worker: the bench configuration at N > 1 (configs[2], weak:
1920x2048 per GPU, RT, walls, 1-D X ring, one process per GPU).

Each rank runs its tile three ways from the same state -- exact single
steps through the peer-store step kernel (the reference's arithmetic, bit
for bit), exact PAIRS through the ring two-step kernel (tlb_peer_step2,
temporal="on"), fast pairs (the bench's headline path) -- and checks on its
own tile: exact pairs == exact single steps bitwise; fast within the
SURVEY §8c contract (f, rho, T <= 1e-12 relative, |du| <= 1e-12 cs).
Ranks agree through an all-reduce; rank 0 prints "FULLSIZE OK".

    python -m torch.distributed.run --nproc-per-node N ... tests/dist_fullsize.py
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    vs = tl.build_velocity_set("D2Q37")
    Lt, Ly, steps = 1920, 2048, 12
    Lx = Lt * world
    tile = tl.decompose(Lx, Ly, world, "1d")[rank]
    macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
    sl = (slice(tile.x0, tile.x0 + Lt), slice(0, Ly))
    f0 = tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(a[sl]), device=dev)
                          for a in macro], vs)

    def advance(arith, temporal):
        p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                             Twall_bot=1.1 * vs.cs2, arith=arith)
        w = tl.RankWorker(tile, vs, p, tl.DistFabric(), schedule="overlapped", device=dev,
                          exchange="p2p", temporal=temporal)
        w.load_block(f0)
        w.run_steps(0, steps)
        out = w.physical_block().clone()
        paired = w.pairable()
        w.collect()
        w.close()
        return out, paired

    exact1, p1 = advance("exact", "off")
    exact2, p2 = advance("exact", "on")
    fast, p3 = advance("fast", "auto")
    ok = (not p1) and p2 and p3
    ok &= bool(torch.equal(exact1, exact2))
    rel_f = ((fast - exact1).abs() / exact1.abs()).max().item()
    mf, me = tl.moments(fast, vs), tl.moments(exact1, vs)
    rel_rho = ((mf[0] - me[0]).abs() / me[0]).max().item()
    rel_T = ((mf[3] - me[3]).abs() / me[3]).max().item()
    du = torch.hypot(mf[1] - me[1], mf[2] - me[2]).max().item() / vs.cs2 ** 0.5
    ok &= max(rel_f, rel_rho, rel_T, du) <= 1e-12
    print(f"rank {rank}: paired {p1} {p2} {p3}, exact pairs == single "
          f"{bool(torch.equal(exact1, exact2))}, fast f {rel_f:.2e} rho {rel_rho:.2e} "
          f"T {rel_T:.2e} |du|/cs {du:.2e}", flush=True)
    flag = torch.tensor([0.0 if ok else 1.0], device=dev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    if rank == 0:
        print("FULLSIZE OK" if flag.item() == 0 else "FULLSIZE FAIL", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
