"""run() throughput on small lattices: CUDA-graph replay vs the per-step
launch loop (timing="every" disables the graphs).

    python tools/small_run.py
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                         arith="exact")
    for (Lx, Ly, steps) in [(256, 128, 2000), (512, 512, 2000), (1920, 2048, 300)]:
        for timing in ("sampled", "every"):
            cfg = tl.SimConfig(Lx=Lx, Ly=Ly, steps=steps, params=p, init="rayleigh-taylor",
                               timing=timing, output="device")
            tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, steps=64, params=p, init="rayleigh-taylor",
                                timing=timing, output="device"))     # warm-up
            t0 = time.perf_counter()
            res = tl.run(cfg)
            el = time.perf_counter() - t0
            print(f"{Lx}x{Ly} steps={steps} timing={timing:8s} "
                  f"{'graphs' if timing != 'every' else 'loop  '} run().mlups={res.mlups:9.1f} "
                  f"us/step={res.wall_seconds / steps * 1e6:8.1f} (call {el:.2f} s)", flush=True)


if __name__ == "__main__":
    main()
