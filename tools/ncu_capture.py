"""Minimal launch sequence for `ncu --set full`: one launch of each step
kernel of interest on the C2 tile (1920x2048, RT, walls), then writes the
SASS hash of each kernel in THIS libtlb.so next to the capture so that
bench.py's ncu_traffic() only trusts a capture of the same binary.

    ncu --set full -k regex:"k_site|k_tb2" -o gpurun_out/X python tools/ncu_capture.py
    python tools/ncu_capture.py --hash-only profiles/<csv>   # writes <csv>.sass
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Lx", type=int, default=1920)
    ap.add_argument("--Ly", type=int, default=2048)
    ap.add_argument("--what", default="single,pair")
    ap.add_argument("--arith", default="fast,exact")
    ap.add_argument("--layout", default="column")
    ap.add_argument("--hash-only", default=None)
    ap.add_argument("--periodic", action="store_true", help="periodic Y instead of walls")
    ap.add_argument("--run", type=int, default=None, help="TLB_TUNE_TB2_RUN")
    ap.add_argument("--cfg", type=int, default=None, help="TLB_TUNE_TB2_CFG for the pair launch")
    ap.add_argument("--init", default="rayleigh-taylor", help="initial condition preset")
    a = ap.parse_args()
    if a.hash_only:
        import bench
        kernels = ["k_tb2<0, 64, 2, 2, 0>", "k_tb2<1, 64, 2, 2, 0>", "k_tb2<0, 64, 2, 2, 1>",
                   "k_tb2<1, 64, 2, 2, 1>", "k_site<3, 0, 4, 0, 4>", "k_site<3, 1, 4, 0, 4>",
                   "k_peer_step<0, 0>", "k_peer_step<1, 0>"]
        with open(a.hash_only + ".sass", "w") as fh:
            for k in kernels:
                fh.write(f"{k} {bench.sass_hash(k)}\n")
        return
    import numpy as np
    import torch
    import paper_1703_00185_b200 as tl
    from paper_1703_00185_b200 import _lib
    from paper_1703_00185_b200.kernels import field_desc
    vs = tl.build_velocity_set("D2Q37")
    _lib.ensure_stencil(vs, 0)
    g = tl.LatticeGeometry(a.Lx, a.Ly, 3, 3, 37, a.layout)
    prv, nxt = tl.allocate_field(g, vs)
    macro = (tl.init.rayleigh_taylor_macro(a.Lx, a.Ly, vs) if a.init == "rayleigh-taylor"
             else tl.init.initial_macro(a.init, a.Lx, a.Ly, vs))
    prv.pops[:, g.phys_x, g.phys_y] = tl.equilibrium(
        *[torch.as_tensor(np.ascontiguousarray(m), device="cuda") for m in macro], vs)
    lib = _lib.load()
    if a.run is not None:
        _lib.check(lib.tlb_set_tuning(3, a.run), "run")
    if a.cfg is not None:
        _lib.check(lib.tlb_set_tuning(2, a.cfg), "cfg")
    st = torch.zeros((2, _lib.STATUS_BYTES), dtype=torch.uint8, device="cuda")
    sp = _lib.stream_ptr()
    for arith in a.arith.split(","):
        tp = _lib.params(tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                                          Twall_bot=1.1 * vs.cs2, arith=arith), vs)
        for what in a.what.split(","):
            if what == "single":
                _lib.check(lib.tlb_step_self(field_desc(prv), field_desc(nxt), tp, int(not a.periodic), int(a.periodic), 1,
                                             st[0].data_ptr(), sp), "step")
            else:
                _lib.check(lib.tlb_step2_self(field_desc(prv), field_desc(nxt), tp, int(not a.periodic), int(a.periodic), 1,
                                              st[0].data_ptr(), st[1].data_ptr(), 0, sp),
                           "step2")
            prv, nxt = nxt, prv
    torch.cuda.synchronize()
    print("ncu_capture done")


if __name__ == "__main__":
    main()
