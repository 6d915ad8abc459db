"""Long-run drift of the fast arithmetic (two steps per launch, the bench
headline path) against the exact arithmetic (bitwise = the reference, so
the GPU exact path stands in for the oracle at step counts the CPU oracle
cannot reach quickly).  Prints, at each checkpoint, the SURVEY §8c contract
quantities: max relative error of f, rho and T, and max |du| / cs.

    python tools/drift_probe.py --Lx 1920 --Ly 2048 --checkpoints 20,100,500,1000
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Lx", type=int, default=1920)
    ap.add_argument("--Ly", type=int, default=2048)
    ap.add_argument("--checkpoints", default="20,100,500,1000")
    a = ap.parse_args()
    vs = tl.build_velocity_set("D2Q37")
    macro = tl.init.rayleigh_taylor_macro(a.Lx, a.Ly, vs)
    f0 = tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(m)).cuda() for m in macro], vs)
    tile = tl.decompose(a.Lx, a.Ly, 1, "1d")[0]
    ws = {}
    for arith in ("fast", "exact"):
        p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                             arith=arith)
        w = tl.RankWorker(tile, vs, p, tl.Fabric(1), schedule="overlapped", layout="column")
        w.load_block(f0)
        ws[arith] = w
    done = 0
    for c in (int(v) for v in a.checkpoints.split(",")):
        for w in ws.values():
            w.run_steps(done, c - done)
            w.collect()
        done = c
        fa, fb = ws["fast"].physical_block(), ws["exact"].physical_block()
        rel_f = float(((fa - fb).abs() / fb.abs()).max())
        ma = tl.moments(fa.reshape(37, -1), vs)
        mb = tl.moments(fb.reshape(37, -1), vs)
        rel_rho = float(((ma[0] - mb[0]).abs() / mb[0]).max())
        rel_T = float(((ma[3] - mb[3]).abs() / mb[3]).max())
        du = float(torch.hypot(ma[1] - mb[1], ma[2] - mb[2]).max()) / float(np.sqrt(vs.cs2))
        print(json.dumps({"lattice": f"{a.Lx}x{a.Ly}", "steps": c, "rel_f": rel_f,
                          "rel_rho": rel_rho, "rel_T": rel_T, "du_over_cs": du,
                          "pairable": ws["fast"].pairable()}), flush=True)


if __name__ == "__main__":
    main()
