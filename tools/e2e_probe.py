"""Phase timing of bench.py's end-to-end paths (host buffers -> K steps ->
host) on the C2 tile, per storage layout.

    python tools/e2e_probe.py [--steps K] [--layouts column,soa]
"""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1703_00185_b200 as tl  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--layouts", default="column,soa,column")
    ap.add_argument("--timing", default="sampled")
    ap.add_argument("--arith", default="exact")
    ap.add_argument("--preload", type=float, default=0.0, help="seconds of steps before rep 0")
    ap.add_argument("--Lx", type=int, default=1920)
    ap.add_argument("--Ly", type=int, default=2048)
    a = ap.parse_args()
    vs = tl.build_velocity_set("D2Q37")
    dev = torch.device("cuda", 0)
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                         arith=a.arith)
    Lx, Ly = a.Lx, a.Ly
    macro = [torch.as_tensor(np.ascontiguousarray(m)).pin_memory()
             for m in tl.init.rayleigh_taylor_macro(Lx, Ly, vs)]
    for layout in a.layouts.split(","):
        tile = tl.decompose(Lx, Ly, 1, "1d")[0]
        w = tl.RankWorker(tile, vs, p, tl.Fabric(1), device=dev, layout=layout,
                          timing=a.timing)
        host_out = torch.empty((37, Lx, Ly), dtype=torch.float64, pin_memory=True)
        import pynvml
        pynvml.nvmlInit()
        hnd = pynvml.nvmlDeviceGetHandleByIndex(0)

        def clocks():
            return (pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_SM),
                    pynvml.nvmlDeviceGetClockInfo(hnd, pynvml.NVML_CLOCK_MEM))
        w.load_block(tl.equilibrium(*[m.to(dev) for m in macro], vs))
        t_end = time.perf_counter() + a.preload
        k = 0
        while time.perf_counter() < t_end:
            for _ in range(20):
                w.step(5000 + k)
                k += 1
            w.synchronize()
            w.collect()
        print(layout, "after preload", k, "steps, clocks", clocks(), flush=True)
        for rep in range(3):
            t = {}
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ts = [m.to(dev, non_blocking=True) for m in macro]
            torch.cuda.synchronize()
            t["h2d_macro"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            f = tl.equilibrium(*ts, vs)
            torch.cuda.synchronize()
            t["equilibrium"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            w.load_block(f)
            torch.cuda.synchronize()
            t["load_block_dev"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(w.stream)
            for s in range(a.steps):
                w.step(1000 * rep + s)
            e1.record(w.stream)
            t["steps_enqueue"] = time.perf_counter() - t0
            t["clk_during"] = clocks()
            torch.cuda.synchronize()
            t["steps"] = time.perf_counter() - t0
            t["steps_device"] = e0.elapsed_time(e1) / 1e3
            t0 = time.perf_counter()
            blk = w.physical_block()
            torch.cuda.synchronize()
            t["physical_block"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            host_out.copy_(blk)
            t["d2h"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            w.load_block(host_out)
            torch.cuda.synchronize()
            t["load_block_host"] = time.perf_counter() - t0
            t0 = time.perf_counter()
            w.collect()
            t["collect"] = time.perf_counter() - t0
            print(layout, rep, {k: (round(v * 1e3, 2) if isinstance(v, float) else v)
                                for k, v in t.items()}, "ms", flush=True)


if __name__ == "__main__":
    main()
