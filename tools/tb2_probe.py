"""Time the two-step kernel (tlb_step2_self) against single fused steps on a
lattice (default C2 1920x2048), CUDA events on the launching stream, after
a ~2 s preload; prints one JSON line per arithmetic.

    python tools/tb2_probe.py [--Lx 1920 --Ly 2048 --steps 200]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib  # noqa: E402
from paper_1703_00185_b200.kernels import field_desc  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Lx", type=int, default=1920)
    ap.add_argument("--Ly", type=int, default=2048)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--arith", default="fast,exact")
    ap.add_argument("--preload", type=float, default=2.0)
    ap.add_argument("--order", default="0", help="work orders (TLB_TUNE_TB2_ORDER)")
    ap.add_argument("--periodic", action="store_true", help="periodic Y instead of walls")
    ap.add_argument("--cfg", default="1", help="two-step kernel shapes to try (TLB_TUNE_TB2_CFG)")
    ap.add_argument("--run", default="0",
                    help="columns per work item (TLB_TUNE_TB2_RUN, 0 = auto)")
    ap.add_argument("--init", default="rayleigh-taylor", help="initial condition preset")
    a = ap.parse_args()
    vs = tl.build_velocity_set("D2Q37")
    _lib.ensure_stencil(vs, 0)
    g = tl.LatticeGeometry(a.Lx, a.Ly, 3, 3, 37, "column")
    prv, nxt = tl.allocate_field(g, vs)
    macro = (tl.init.rayleigh_taylor_macro(a.Lx, a.Ly, vs) if a.init == "rayleigh-taylor"
             else tl.init.initial_macro(a.init, a.Lx, a.Ly, vs))
    prv.pops[:, g.phys_x, g.phys_y] = tl.equilibrium(
        *[torch.as_tensor(np.ascontiguousarray(m), device="cuda") for m in macro], vs)
    lib = _lib.load()
    st = torch.zeros((2, _lib.STATUS_BYTES), dtype=torch.uint8, device="cuda")
    sp = _lib.stream_ptr()
    sites = a.Lx * a.Ly
    wl, pe = (0, 1) if a.periodic else (1, 0)
    for arith in a.arith.split(","):
        p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                             Twall_bot=1.1 * vs.cs2, arith=arith)
        tp = _lib.params(p, vs)
        bufs = [prv, nxt]

        def one(n):
            for _ in range(n):
                _lib.check(lib.tlb_step_self(field_desc(bufs[0]), field_desc(bufs[1]), tp, wl, pe,
                                             1, st[0].data_ptr(), sp), "step")
                bufs.reverse()

        def two(n):
            for _ in range(n // 2):
                _lib.check(lib.tlb_step2_self(field_desc(bufs[0]), field_desc(bufs[1]), tp, wl, pe,
                                              1, st[0].data_ptr(), st[1].data_ptr(), 0, sp),
                           "step2")
                bufs.reverse()

        res = {"arith": arith, "Lx": a.Lx, "Ly": a.Ly, "steps": a.steps}
        variants = [("single", one, None)]
        for cfg in a.cfg.split(","):
            for run in a.run.split(","):
                for order in a.order.split(","):
                    variants.append((f"two_cfg{cfg}_run{run}_o{order}", two,
                                     (int(cfg), int(run), int(order))))
        variants.append(("single_again", one, None))
        for name, fn, tune in variants:
            if tune:
                _lib.check(lib.tlb_set_tuning(2, tune[0]), "cfg")
                _lib.check(lib.tlb_set_tuning(3, tune[1]), "run")
                _lib.check(lib.tlb_set_tuning(4, tune[2]), "order")
            fn(10)
            torch.cuda.synchronize()
            t0 = time.time()
            while time.time() - t0 < a.preload:
                fn(20)
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn(a.steps)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.steps
            res[name] = {"ms_per_step": round(ms, 5), "mlups": round(sites / ms / 1e3, 1)}
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
