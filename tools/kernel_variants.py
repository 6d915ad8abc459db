"""Time fused-kernel variants on the C2 tile (1920x2048) with CUDA events.

    python tools/kernel_variants.py [--reps N]

Used to attribute the fused step's cost (implicit halos, wall rows, exact vs
fast arithmetic) before and after kernel changes; numbers go to profiles/.
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--Lx", type=int, default=1920)
    ap.add_argument("--Ly", type=int, default=2048)
    ap.add_argument("--only", default="")
    ap.add_argument("--pad", type=int, default=0,
                    help="align: column pitch multiple of 16 doubles, y=Hy at a 128 B boundary")
    ap.add_argument("--layout", default="column", choices=["column", "soa", "aos"])
    a = ap.parse_args()
    vs = tl.build_velocity_set("D2Q37")
    g = tl.LatticeGeometry(a.Lx, a.Ly, 3, 3, 37, "soa" if a.pad else a.layout)
    prv, nxt = tl.allocate_field(g, vs)
    if a.pad:
        # same logical (Q, NX, NY) view over a padded, 128 B aligned allocation
        off = (16 - g.Hy % 16) % 16
        pitch = -(-(g.NY + off) // 16) * 16
        for fld in (prv, nxt):
            buf = torch.zeros((37, g.NX, pitch), dtype=torch.float64, device="cuda")
            fld.data = buf[:, :, off:off + g.NY]
        print(f"padded: pitch {pitch}, offset {off}", flush=True)
    macro = tl.init.rayleigh_taylor_macro(a.Lx, a.Ly, vs)
    f0 = tl.equilibrium(*[torch.as_tensor(m).cuda() for m in macro], vs)
    prv.pops[:, g.phys_x, g.phys_y] = f0
    nxt.pops.copy_(prv.pops)
    lib = _lib.load()
    st = _lib.Status(prv.device)
    s = torch.cuda.current_stream().cuda_stream
    P, N = field_desc(prv), field_desc(nxt)
    full = _lib.region(g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly)
    ex = _lib.params(tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                                      Twall_bot=1.1 * vs.cs2))
    fa = _lib.params(tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                                      Twall_bot=1.1 * vs.cs2, arith="fast"))
    W = _lib.F_WALL_BOT | _lib.F_WALL_TOP
    IMP = _lib.F_CLAMP_Y | _lib.F_WRAP_X
    variants = {
        "propagate": lambda: lib.tlb_propagate(P, N, full, s),
        "collide_exact_inplace": lambda: lib.tlb_collide(N, N, full, ex, 0, st.ptr, s),
        "collide_exact_oop": lambda: lib.tlb_collide(P, N, full, ex, 0, st.ptr, s),
        "collide_fast_inplace": lambda: lib.tlb_collide(N, N, full, fa, 0, st.ptr, s),
        "fused_exact_plain": lambda: lib.tlb_fused(P, N, full, ex, 0, st.ptr, s),
        "fused_exact_walls": lambda: lib.tlb_fused(P, N, full, ex, W, st.ptr, s),
        "fused_exact_step": lambda: lib.tlb_fused(P, N, full, ex, W | IMP, st.ptr, s),
        "fused_exact_step_neg": lambda: lib.tlb_fused(P, N, full, ex, W | IMP | _lib.F_COUNT_NEG,
                                                      st.ptr, s),
        "fused_fast_plain": lambda: lib.tlb_fused(P, N, full, fa, 0, st.ptr, s),
        "fused_fast_step": lambda: lib.tlb_fused(P, N, full, fa, W | IMP, st.ptr, s),
        "fused_fast_walls": lambda: lib.tlb_fused(P, N, full, fa, W, st.ptr, s),
        "fused_fast_wrap": lambda: lib.tlb_fused(P, N, full, fa, _lib.F_WRAP_X, st.ptr, s),
    }
    def tuned(fn, key, val, default):
        def run():
            lib.tlb_set_tuning(key, val)
            r = fn()
            lib.tlb_set_tuning(key, default)
            return r
        return run
    for mb in (1, 5):
        variants[f"fused_exact_step_neg_minb{mb}"] = tuned(variants["fused_exact_step_neg"], 1, mb, 4)
        variants[f"fused_fast_step_minb{mb}"] = tuned(variants["fused_fast_step"], 1, mb, 4)
    sites = a.Lx * a.Ly
    out = {}
    order = a.only.split(",") if a.only else list(variants)   # --only order, repeats allowed
    for name in order:
        fn = variants[name]
        ts = []
        for _ in range(a.reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(fn(), name)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts[1:]))
        out[name] = {"ms": round(ms, 4), "GBps_592": round(592 * sites / ms / 1e6, 1),
                     "mlups": round(sites / ms / 1e3, 1)}
        print(f"{name:24s} {ms:8.4f} ms  {592 * sites / ms / 1e6:8.1f} GB/s  "
              f"{sites / ms / 1e3:8.1f} MLUPS", flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
