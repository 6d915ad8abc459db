"""Small lattices (C1 256x128, ...): device time per step of the launch
policies, CUDA events around 32-step blocks after a warm-up.

    python tools/small_probe.py [--sizes 256x128,512x256] [--reps 20]

site_graph  : single-step fused kernel k_site, 32 launches in a CUDA graph
pairs_graph : the two-step kernel, 16 launches in a CUDA graph
(the persistent multi-step, split-site and loop-rolled kernels measured in
round 2 live on the exp/small-tiles branch; profiles/r02_small.md)
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
    ap.add_argument("--sizes", default="256x128,512x256")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    lib = _lib.load()
    vs = tl.build_velocity_set("D2Q37")
    _lib.ensure_stencil(vs, 0)
    K = 32
    st = torch.zeros((K, _lib.STATUS_BYTES), dtype=torch.uint8, device="cuda")
    sp = lambda: torch.cuda.current_stream().cuda_stream  # noqa: E731
    for size in a.sizes.split(","):
        Lx, Ly = (int(v) for v in size.split("x"))
        g = tl.LatticeGeometry(Lx, Ly, 3, 3, 37, "column")
        prv, nxt = tl.allocate_field(g, vs)
        macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
        prv.pops[:, g.phys_x, g.phys_y] = tl.equilibrium(
            *[torch.as_tensor(np.ascontiguousarray(m), device="cuda") for m in macro], vs)
        for arith in ("exact", "fast"):
            tp = _lib.params(tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                                              Twall_bot=1.1 * vs.cs2, arith=arith), vs)
            A, B = field_desc(prv), field_desc(nxt)

            def site_step(k):
                _lib.check(lib.tlb_step_self(A if k % 2 == 0 else B, B if k % 2 == 0 else A,
                                             tp, 1, 0, 1, st[k].data_ptr(), sp()), "step")

            def pair(k):
                _lib.check(lib.tlb_step2_self(A if k % 2 == 0 else B, B if k % 2 == 0 else A,
                                              tp, 1, 0, 1, st[k].data_ptr(), st[k + 1].data_ptr(),
                                              k, sp()), "step2")

            def graph_of(fn, stride):
                for k in range(0, K, stride):   # warm-up (allocations) outside capture
                    fn(k)
                torch.cuda.synchronize()
                gr = torch.cuda.CUDAGraph()
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    gr.capture_begin()
                    for k in range(0, K, stride):
                        fn(k)
                    gr.capture_end()
                torch.cuda.synchronize()
                return gr.replay

            policies = {
                "site_graph": graph_of(site_step, 1),
                "pairs_graph": graph_of(pair, 2),
            }
            for name, fn in policies.items():
                for _ in range(3):
                    fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.reps):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3 / (a.reps * K)
                print(json.dumps({"lattice": size, "arith": arith, "policy": name,
                                  "us_per_step": round(us, 2),
                                  "mlups": round(Lx * Ly / us, 1)}), flush=True)


if __name__ == "__main__":
    main()
