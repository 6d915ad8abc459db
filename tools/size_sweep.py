"""Fused-step bandwidth vs lattice size and q-plane stride.

    python tools/size_sweep.py [--reps N]

Why does the C2 tile (1920x2048) reach ~93 % of the measured HBM copy rate
while 4096x8192 reaches ~98 %?  For each size this times the fused fast step
(and, for scale, a torch copy of the same 2 x 296 B/site) with the q-plane
stride as allocated and padded by a few KB (to break any plane aliasing in
the HBM channel hash).  Output: one line per case, JSON at the end.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib  # noqa: E402
from paper_1703_00185_b200.kernels import field_desc  # noqa: E402


def timeit(fn, reps):
    ts = []
    for _ in range(reps + 2):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts[2:]))


def fields(g, pad, layout="soa"):
    out = []
    for _ in range(2):
        if layout == "xqy":   # (NX, Q, NY) storage viewed as (Q, NX, NY)
            buf = torch.zeros(37 * g.NX * g.NY, dtype=torch.float64, device="cuda")
            out.append(buf.as_strided((37, g.NX, g.NY), (g.NY, 37 * g.NY, 1)))
            continue
        sl = g.NX * g.NY + pad
        buf = torch.zeros(37 * sl, dtype=torch.float64, device="cuda")
        out.append(buf.as_strided((37, g.NX, g.NY), (sl, g.NY, 1)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--sizes", default="1920x2048,1920x4096,3840x2048,3840x4096,4096x8192")
    ap.add_argument("--pads", default="0,1040")
    ap.add_argument("--layouts", default="soa")
    a = ap.parse_args()
    vs = tl.build_velocity_set("D2Q37")
    lib = _lib.load()
    st = _lib.Status(torch.device("cuda", 0))
    s = torch.cuda.current_stream().cuda_stream
    fa = _lib.params(tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                                      Twall_bot=1.1 * vs.cs2, arith="fast"))
    flags = _lib.F_WALL_BOT | _lib.F_WALL_TOP | _lib.F_CLAMP_Y | _lib.F_WRAP_X
    res = {}
    for size in a.sizes.split(","):
        Lx, Ly = (int(v) for v in size.split("x"))
        g = tl.LatticeGeometry(Lx, Ly, 3, 3, 37)
        macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
        f0 = tl.equilibrium(*[torch.as_tensor(m).cuda() for m in macro], vs)
        sites = Lx * Ly
        cases = [(lay, int(p)) for lay in a.layouts.split(",")
                 for p in (a.pads.split(",") if lay == "soa" else ["0"])]
        for lay, pad in cases:
            prv, nxt = fields(g, pad, lay)
            prv[:, 3:3 + Lx, 3:3 + Ly] = f0
            P = _lib.field(prv, Lx, Ly, 3, 3)
            N = _lib.field(nxt, Lx, Ly, 3, 3)
            full = _lib.region(3, 3 + Lx, 3, 3 + Ly)
            ms = timeit(lambda: lib.tlb_fused(P, N, full, fa, flags, st.ptr, s), a.reps)
            key = f"{size}/{lay}/pad{pad}"
            res[key] = {"fused_ms": round(ms, 4), "GBps": round(592 * sites / ms / 1e6, 1)}
            del prv, nxt
            torch.cuda.empty_cache()
        src = torch.empty(37 * sites, dtype=torch.float64, device="cuda")
        dst = torch.empty_like(src)
        ms = timeit(lambda: dst.copy_(src), a.reps)
        res[f"{size}/copy"] = {"ms": round(ms, 4), "GBps": round(592 * sites / ms / 1e6, 1)}
        del src, dst, f0
        torch.cuda.empty_cache()
        for k, v in res.items():
            if k.startswith(size + "/"):
                print(f"{k:24s} {v}", flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
