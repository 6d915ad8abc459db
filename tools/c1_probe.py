"""Small lattices through run(): per-step device time of each launch policy.

    python tools/c1_probe.py [--steps 2048]

graph = single steps replayed from a CUDA graph (temporal off); pairs =
two-step kernel launches; auto = run()'s default choice.  Device time per step from the launch events
(t_bulk) and wall time per step of run(); one JSON line per case.
"""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2048)
    ap.add_argument("--sizes", default="256x128,512x256,1024x512")
    a = ap.parse_args()
    vs = tl.build_velocity_set("D2Q37")
    policies = {"graph": dict(temporal="off"), "pairs": dict(temporal="on"),
                "auto": dict()}
    for arith in ("exact", "fast"):
        p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                             arith=arith)
        for size in a.sizes.split(","):
            Lx, Ly = (int(v) for v in size.split("x"))
            for name, kw in policies.items():
                base = dict(Lx=Lx, Ly=Ly, params=p, init="rayleigh-taylor", output="device", **kw)
                tl.run(tl.SimConfig(steps=64, **base))
                r = tl.run(tl.SimConfig(steps=a.steps, **base))
                tb = np.array([m["t_bulk"] for m in r.metrics])
                dev_us = float(np.nanmean(tb)) * 1e6
                print(json.dumps({"arith": arith, "lattice": size, "policy": name,
                                  "steps": a.steps,
                                  "wall_us_per_step": round(r.wall_seconds / a.steps * 1e6, 2),
                                  "device_us_per_step": round(dev_us, 2),
                                  "mlups_wall": round(r.mlups, 1),
                                  "mlups_device": round(Lx * Ly / dev_us, 1)}), flush=True)


if __name__ == "__main__":
    main()
