"""D2Q9 through the generic kernels: per-step device time on large tiles vs
its own roofline (9 + 9 doubles = 144 B per site update).

    python tools/d2q9_rate.py
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    vs = tl.build_velocity_set("D2Q9")
    dev = torch.device("cuda", 0)
    for Lx, Ly in ((1920, 2048), (4096, 8192)):
        p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
        tile = tl.decompose(Lx, Ly, 1, "1d")[0]
        w = tl.RankWorker(tile, vs, p, tl.Fabric(1), schedule="overlapped", device=dev,
                          timing="off")
        macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
        w.load_block(tl.equilibrium(*[torch.as_tensor(m, device=dev) for m in macro], vs))
        K = 50
        for rep in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(w.stream)
            for s in range(K):
                w.step(1000 * rep + s)
            e1.record(w.stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / K
            w.collect()
        print(f"D2Q9 {Lx}x{Ly}: {ms * 1e3:.1f} us/step, {Lx * Ly / ms / 1e3:.0f} MLUPS, "
              f"{144 * Lx * Ly / ms / 1e6:.0f} GB/s (144 B/site)", flush=True)
        del w


if __name__ == "__main__":
    main()
