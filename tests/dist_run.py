"""torchrun worker for the multi-GPU tests (one process per GPU, NCCL).

    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 \
        --master-port P tests/dist_run.py

Runs sim.run with Np = world size (1-D X tiling, X faces exchanged over
NCCL) for both schedules and compares the gathered state with the C oracle
(bitwise, exact arithmetic) on rank 0.  Prints "DIST OK" on success.
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
    local = int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gx=2e-6, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                         Twall_bot=1.1 * vs.cs2)
    Lx, Ly, steps = 48 * world, 40, 9
    want = None
    if rank == 0:
        from oracle import oracle as O
        O.set_stencil(vs.c, vs.w, vs.cs2)
        f0 = O.equilibrium(*O.rayleigh_taylor_macro(Lx, Ly, vs.cs2))
        p6 = O.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top, p.Twall_bot)
        want, neg = O.run(f0, steps, p6)
        want_periodic, _ = O.run(f0, steps, p6, ymode="periodic")
    tilings = ["1d", (1, world)] + ([(2, world // 2)] if world >= 4 else [])
    cases = [(t, sch, "nccl") for t in tilings for sch in ("overlapped", "staged")]
    cases.append(("1d", "overlapped", "p2p"))      # NVLink peer-store exchange
    cases.append(("1d", "overlapped", "auto"))     # the default (p2p where it applies)
    cases.append(((1, world), "overlapped", "p2p"))  # Y split only: X self-periodic
    if world >= 4:
        cases.append(((2, world // 2), "overlapped", "p2p"))   # 2-D: corners diagonal
    cases = [c + (False,) for c in cases]
    # periodic Y: up/down neighbours wrap (2-D: the same rank above and below)
    cases.append(((1, world), "overlapped", "p2p", True))
    if world >= 4:
        cases.append(((2, world // 2), "overlapped", "p2p", True))
        cases.append(((2, world // 2), "overlapped", "nccl", True))
    ok = True
    # snapshots (reduced to rho, u, T on the device and gathered on rank 0,
    # reference sim.py:89-90, 119-125) and NaN-poisoned halos (runtime.py:
    # 288-294) on both native transports
    for exchange in ("p2p", "nccl"):
        res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=world, steps=steps, params=p,
                                  init="rayleigh-taylor", exchange=exchange,
                                  snapshot_every=3, debug_poison=True))
        if rank == 0:
            same = np.array_equal(res.populations, want)
            snaps_ok = [s for s, _ in res.snapshots] == [3, 6, 9]
            for s_, m in res.snapshots:
                ref_s, _ = O.run(f0, s_, p6)
                rho, ux, uy, T = O.moments(ref_s)
                snaps_ok &= all(np.array_equal(a, b) for a, b in
                                ((m.rho, rho), (m.ux, ux), (m.uy, uy), (m.T, T)))
            rho, ux, uy, T = O.moments(want)
            macro_ok = np.array_equal(res.macro.rho, rho) and np.array_equal(res.macro.T, T)
            print(f"snapshots+poison exchange={exchange} world={world} ok={same} "
                  f"snapshots={snaps_ok} macro={macro_ok}", flush=True)
            ok &= same and snaps_ok and macro_ok
    for tiling, schedule, exchange, periodic in cases:
        for arith in (("exact", "fast") if exchange == "p2p" else ("exact",)):
            pp = tl.PhysicsParams(tau=p.tau, gx=p.gx, gy=p.gy, Twall_top=p.Twall_top,
                                  Twall_bot=p.Twall_bot, arith=arith)
            res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=world, tiling=tiling, steps=steps,
                                      params=pp, init="rayleigh-taylor", schedule=schedule,
                                      exchange=exchange, walls=not periodic,
                                      periodic_y=periodic))
            if rank == 0:
                ref = want_periodic if periodic else want
                if arith == "exact":
                    same = np.array_equal(res.populations, ref)
                else:
                    same = bool(np.max(np.abs(res.populations - ref) / np.abs(ref)) < 1e-12)
                print(f"tiling={tiling} schedule={schedule} exchange={exchange} arith={arith} "
                      f"periodic={periodic} world={world} ok={same} mlups={res.mlups:.1f}",
                      flush=True)
                ok &= same
            assert len(res.metrics) == steps
    # two steps per launch across the GPUs (tlb_peer_step2 over CUDA IPC):
    # walls and periodic Y, an odd step count (a final single step) and
    # snapshots between pairs
    for periodic in (False, True):
        for arith in ("exact", "fast"):
            pp = tl.PhysicsParams(tau=p.tau, gx=p.gx, gy=p.gy, Twall_top=p.Twall_top,
                                  Twall_bot=p.Twall_bot, arith=arith)
            res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=world, steps=steps, params=pp,
                                      init="rayleigh-taylor", exchange="p2p", temporal="on",
                                      walls=not periodic, periodic_y=periodic,
                                      snapshot_every=4))
            if rank == 0:
                ref = want_periodic if periodic else want
                if arith == "exact":
                    same = np.array_equal(res.populations, ref)
                else:
                    same = bool(np.max(np.abs(res.populations - ref) / np.abs(ref)) < 1e-12)
                same &= [s for s, _ in res.snapshots] == [4, 8]
                print(f"pairs exchange=p2p arith={arith} periodic={periodic} world={world} "
                      f"ok={same} mlups={res.mlups:.1f}", flush=True)
                ok &= same
            assert len(res.metrics) == steps
    # 6-wide halos (what a ring rank that pairs steps allocates) on the NCCL
    # ring and the single-step peer kernel: the halo width is a parameter
    for exchange in ("nccl", "p2p"):
        res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=world, steps=steps, params=p,
                                  init="rayleigh-taylor", exchange=exchange, halo=6))
        if rank == 0:
            same = np.array_equal(res.populations, want)
            print(f"halo=6 exchange={exchange} world={world} ok={same}", flush=True)
            ok &= same
    dist.barrier()
    if rank == 0:
        print("DIST OK" if ok else "DIST FAIL", flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
