#!/usr/bin/env python
"""D2Q37 thermal-LBM time-step benchmark (BASELINE.json metric).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

A "step" is one full time step (X-halo exchange + propagate + bc + collide,
fused) of the whole lattice.  At N=1 the workload is BASELINE.json configs[1]
(D2Q37 Rayleigh-Taylor 1920x2048 on one B200); at N>1 it is configs[2]
(weak scaling, 1920x2048 per GPU, 1-D X tiling; the X halos travel as
NVLink peer stores fused into the step kernel, or over an overlapped NCCL
ring with --exchange nccl), one process per GPU under torchrun; --strong
gives configs[3].  Prints ONE JSON line on rank 0.

--impl reference times the reference algorithm on the host CPU (the C
oracle restatement, all host threads) on a bounded sample of the workload.
"""

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MLUPS and FP64 sustained GFLOPS per step at 1/2/4/8 B200 vs roofline and CPU ref"
FLOP_SITE = 2764          # collide, algorithmic
FLOP_WALL_SITE = 2449     # bc, per wall-row site
BYTES_SITE = 592          # fused step: 37 x 8 B read + 37 x 8 B written
TILE_LX, TILE_LY = 1920, 2048


_SASS = None


def sass_hash(kernel):
    """sha256 (16 hex) of the SASS of the libtlb.so function whose demangled
    name contains `kernel` (cuobjdump), or None."""
    global _SASS
    import hashlib
    import re
    if _SASS is None:
        lib = os.path.join(ROOT, "paper_1703_00185_b200", "libtlb.so")
        try:
            txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True,
                                 timeout=120).stdout
            dem = subprocess.run(["cu++filt"], input="\n".join(
                re.findall(r"Function : (\S+)", txt)), capture_output=True, text=True,
                timeout=60).stdout.split("\n")
        except (OSError, subprocess.SubprocessError):
            _SASS = {}
            return None
        blocks = re.split(r"\n\s*Function : \S+", txt)[1:]
        _SASS = dict(zip(dem, blocks))
    for name, body in _SASS.items():
        if kernel in name.replace("(bool)", "").replace("(int)", ""):
            # drop addresses and encodings: the instruction text only
            ins = re.findall(r"/\*[0-9a-f]{4,}\*/\s+([^;]*;)", body)
            return hashlib.sha256("\n".join(ins).encode()).hexdigest()[:16]
    return None


def ncu_traffic(kernel, layout="column"):
    """dram__bytes_read.sum + dram__bytes_write.sum (GB) of `kernel` from the
    committed `ncu --set full` capture of the same storage layout
    (profiles/*ncu*_<layout>_raw*.csv) -- only from a capture whose sidecar
    <csv>.sass records the SASS hash of the kernel in THIS libtlb.so."""
    import csv
    import glob
    want_hash = sass_hash(kernel)
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"*ncu*_{layout}_raw*.csv")),
                   reverse=True)
    for path in paths:
        try:
            with open(path + ".sass") as fh:
                tags = dict(line.strip().rsplit(" ", 1) for line in fh if " " in line)
            rows = list(csv.reader(open(path)))
        except (OSError, ValueError):
            continue
        if not rows or want_hash is None or tags.get(kernel) != want_hash:
            continue
        hdr = rows[0]
        for r in rows[2:]:
            d = dict(zip(hdr, r))
            if kernel in d.get("Kernel Name", "").replace("(bool)", "").replace("(int)", ""):
                try:
                    return round(float(d["dram__bytes_read.sum"]) +
                                 float(d["dram__bytes_write.sum"]), 4), \
                        f"{os.path.basename(path)} (SASS {want_hash})"
                except (KeyError, ValueError):
                    continue
    return None, f"no capture of this binary's {kernel} (SASS {want_hash})"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


# ----------------------------------------------------------------- clocks --

class ClockSampler:
    """nvidia-smi sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap,utilization.gpu")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, gpu_id):
        self.gpu_id = gpu_id
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100", "-i", str(self.gpu_id)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi can take seconds to start on a multi-GPU box: wait for
            # its first sample so the load phase is actually observed
            t0 = time.time()
            while not self.rows and time.time() - t0 < 15 and self.proc.poll() is None:
                time.sleep(0.05)
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        def parse(rows, loaded_only):
            sm, smax, reasons = [], [], set()
            for r in rows:
                try:
                    util = float(r[7])
                except ValueError:
                    util = 100.0
                try:
                    power = float(r[2])
                except ValueError:
                    power = 1000.0
                if loaded_only and util < 50 and power < 300:
                    continue
                try:
                    sm.append(float(r[0]))
                    smax.append(float(r[1]))
                except ValueError:
                    continue
                for name, v in zip(self.NAMES, r[3:7]):
                    if v.lower() == "active":
                        reasons.add(name)
            return sm, smax, reasons

        sm, smax, reasons = parse(self.rows, True)
        loaded = bool(sm)
        if not sm:  # no sample classified as under load: report all of them
            sm, smax, reasons = parse(self.rows, False)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "samples_total": len(self.rows)}
        power = []
        for r in self.rows:
            try:
                power.append(float(r[2]))
            except ValueError:
                pass
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(smax),
                "reasons": sorted(reasons), "samples": len(sm),
                "samples_total": len(self.rows), "under_load": loaded,
                "power_w_median": float(np.median(power)) if power else None}


# ------------------------------------------------------------ CPU oracle --

def _oracle_setup():
    from oracle import oracle as O
    import paper_1703_00185_b200 as tl
    O.build()
    vs = tl.build_velocity_set("D2Q37")
    O.set_stencil(vs.c, vs.w, vs.cs2)
    nthreads = len(os.sched_getaffinity(0))
    O.threads(nthreads)
    p6 = O.params6(0.8, 0.0, -1e-5, 1.0, 0.9 * vs.cs2, 1.1 * vs.cs2)
    return O, vs, nthreads, p6


def cpu_oracle_rate(seconds=None, steps=None, warmup=2, Lx=TILE_LX, Ly=TILE_LY):
    """The C oracle (oracle/tlb_oracle.c, bitwise = the reference) with all
    host threads on the RT Lx x Ly lattice itself: `warmup` untimed steps
    (OpenMP pool up, buffers faulted in), then `steps` steps -- or as many as
    fit in `seconds`, sized from a one-step probe -- timed inside the C
    library.  Returns (MLUPS, threads, steps, seconds, description)."""
    O, vs, nthreads, p6 = _oracle_setup()
    f0 = O.equilibrium(*O.rayleigh_taylor_macro(Lx, Ly, vs.cs2))
    if steps is None:
        _, one = O.run_timed(f0, 1, 1, p6)
        steps = max(3, int(seconds / max(one, 1e-6)))
    _, el = O.run_timed(f0, warmup, steps, p6)
    return (Lx * Ly * steps / el / 1e6, nthreads, steps, el,
            f"RT {Lx}x{Ly} (walls, periodic X), {warmup} untimed + {steps} timed steps, "
            f"{nthreads} threads, {el:.2f} s")


def numpy_reference_rates(budget_s=60.0):
    """The reference package itself (`thermolb`, pip-installed from
    /root/reference into baseline/_ref, which travels to the GPU box) timed
    through its public run() (sim.py:62-129; MLUPS = Lx*Ly*steps/wall,
    :127) as SURVEY §8(d) asks: C1 RT 256x128 at Np=1 (numpy ufuncs are
    single-threaded: one core) and C2 RT 1920x2048 at Np = the host cores
    (1-D tiles on worker threads; numpy releases the GIL), 2 steps.
    Returns a dict, or {"unavailable": why}."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "thermolb")):
        return {"unavailable": "baseline/_ref not installed (see DESIGN.md)"}
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import thermolb
        from thermolb import PhysicsParams, SimConfig, build_velocity_set, run
    except Exception as e:  # noqa: BLE001 -- report, do not fail the arm
        return {"unavailable": f"import thermolb failed: {e!r}"[:200]}
    vs = build_velocity_set("D2Q37")
    p = PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    cores = len(os.sched_getaffinity(0))
    np_c2 = max(d for d in range(1, cores + 1) if TILE_LX % d == 0)
    out = {"package": f"thermolb {thermolb.__version__} (baseline/_ref)",
           "api": "thermolb.run(SimConfig) (sim.py:62-129)"}
    t_start = time.time()
    for name, Lx, Ly, Np, steps in (("C1", 256, 128, 1, 100), ("C2", TILE_LX, TILE_LY, np_c2, 2)):
        if time.time() - t_start > budget_s:
            out[name] = {"skipped": f"over the {budget_s:.0f} s budget"}
            continue
        cfg = SimConfig(Lx=Lx, Ly=Ly, Np=Np, tiling="1d", schedule="overlapped", steps=steps,
                        params=p, init="rayleigh-taylor")
        res = run(cfg)
        out[name] = {"lattice": f"{Lx}x{Ly}", "Np": Np, "cores": Np, "steps": steps,
                     "wall_s": round(res.wall_seconds, 3), "mlups": round(res.mlups, 4),
                     "gflops_fp64": round(res.mlups * FLOP_SITE / 1e3, 3)}
    # the reference's kernels one by one on one core (SURVEY §8d "per-kernel
    # split on C2"): propagate and bc over the whole C2 tile, collide on a
    # 240-column band of it (the same per-site work; ~1/8 of the ~21 s a
    # full C2 collide takes) scaled to the tile
    if time.time() - t_start < budget_s:
        try:
            from thermolb import allocate_field, bc, collide, propagate
            from thermolb.geometry import LatticeGeometry
            from thermolb.init import build_initial_state
            g = LatticeGeometry(TILE_LX, TILE_LY, 3, 3, vs.Q)
            prv, nxt = allocate_field(g, vs)
            prv.pops[:, g.phys_x, g.phys_y] = build_initial_state("rayleigh-taylor", TILE_LX,
                                                                   TILE_LY, vs)
            sites = TILE_LX * TILE_LY
            t0 = time.perf_counter()
            propagate(prv, nxt, vs)
            t_prop = time.perf_counter() - t0
            t0 = time.perf_counter()
            bc(nxt, p, vs)
            t_bc = time.perf_counter() - t0
            band = nxt.pops[:, g.Hx:g.Hx + 240, g.phys_y]
            t0 = time.perf_counter()
            collide(band, p, vs)
            t_col = (time.perf_counter() - t0) * TILE_LX / 240
            out["split_C2_1core"] = {
                "propagate_s": round(t_prop, 4), "bc_s": round(t_bc, 4),
                "collide_s": round(t_col, 3), "collide_sample": "240x2048 band, scaled x8",
                "propagate_GBps": round(BYTES_SITE * sites / t_prop / 1e9, 3),
                "collide_gflops": round(FLOP_SITE * sites / t_col / 1e9, 3)}
        except Exception as e:  # noqa: BLE001 -- report, do not fail the arm
            out["split_C2_1core"] = {"unavailable": repr(e)[:200]}
    return out


def reference_arm(args, rank, world):
    """--impl reference: the reference algorithm on the host CPU (the C
    oracle, every host thread) on the workload of the GPU arm's config --
    configs[1]/[2]: the whole (1920*N) x 2048 lattice, W untimed + K timed
    steps; configs[3] (strong, 8192x16384 = 79.5 GB of host buffers): a
    1024x16384 column band of it, the per-site work being identical."""
    if rank != 0:
        return 0
    if args.strong:
        Lx, Ly = 8192, 16384
        sLx, sLy = 1024, 16384
        workload = f"D2Q37 RT {Lx}x{Ly} (strong scaling, {world} tiles)"
    else:
        Lx, Ly = args.Lx * world, args.Ly
        sLx, sLy = Lx, Ly
        workload = (f"D2Q37 RT {Lx}x{Ly} on 1 B200 (BASELINE configs[1])" if world == 1 else
                    f"D2Q37 RT {Lx}x{Ly} (1-D X tiles of {args.Lx}x{args.Ly})")
    mlups, nthreads, done, el, sample = cpu_oracle_rate(steps=args.steps, warmup=args.warmup,
                                                        Lx=sLx, Ly=sLy)
    ms_step = el / done * 1e3 * (Lx * Ly) / (sLx * sLy)
    line = {
        "impl": "reference", "metric": METRIC, "value": round(mlups, 4), "unit": "MLUPS",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3),
        "higher_is_better": True, "scaling": "strong" if args.strong else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (Rayleigh-Taylor init)",
        "config": {"workload": workload, "sample": sample,
                   "same_lattice": (sLx, sLy) == (Lx, Ly)},
        "gflops_fp64": round(mlups * FLOP_SITE / 1e3, 3),
        "cpu_baseline": {"value": round(mlups, 4), "unit": "MLUPS", "cores": nthreads,
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(mlups, 4), "unit": "MLUPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    if args.numpy_ref:
        line["numpy_reference"] = numpy_reference_rates()
    emit(line)
    return 0


# --------------------------------------------------------------- GPU arm --

def gpu_arm(args, rank, world, local_rank):
    import torch
    import paper_1703_00185_b200 as tl
    from paper_1703_00185_b200 import _lib
    from paper_1703_00185_b200.kernels import field_desc

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    vs = tl.build_velocity_set("D2Q37")
    grid = (world, 1)
    if args.tiling != "1d":
        grid = tuple(int(v) for v in args.tiling.lower().split("x"))
        if grid[0] * grid[1] != world:
            raise SystemExit(f"--tiling {args.tiling} does not match {world} ranks")
    if args.strong:
        # BASELINE configs[3]: fixed 8192x16384 lattice split over the GPUs
        Lx, Ly = 8192, 16384
        Lx_tile, Ly_tile = Lx // grid[0], Ly // grid[1]
    else:
        Lx_tile, Ly_tile = args.Lx, args.Ly
        Lx, Ly = Lx_tile * grid[0], Ly_tile * grid[1]
    p = tl.PhysicsParams(tau=0.8, gx=0.0, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                         Twall_bot=1.1 * vs.cs2, arith=args.arith)
    if args.tb2_order != -1:
        _lib.check(_lib.load().tlb_set_tuning(4, args.tb2_order), "tb2 order")
    tiles = tl.decompose(Lx, Ly, world, "1d" if grid[1] == 1 else grid)
    tile = tiles[rank]
    fabric = tl.DistFabric() if world > 1 else tl.Fabric(1)
    w = tl.RankWorker(tile, vs, p, fabric, schedule=args.schedule, device=dev,
                      exchange=args.exchange, layout=args.layout)
    macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
    sl = (slice(tile.x0, tile.x0 + Lx_tile), slice(tile.y0, tile.y0 + Ly_tile))
    f0 = tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(a[sl]), device=dev)
                          for a in macro], vs)
    w.load_block(f0)
    torch.cuda.synchronize()

    def barrier():
        if dist is not None:
            dist.barrier(device_ids=[local_rank])

    # one tile (N=1): two steps per launch where it applies (temporal
    # blocking, csrc/tb2.cu; RankWorker.pairable) -- run()'s own path
    def run_steps(n, s0=0):
        pair = w.pairable()
        s = s0
        while s < s0 + n:
            if pair and s + 1 < s0 + n:
                w.step_pair(s)
                s += 2
            else:
                w.step(s)
                s += 1

    # warm-up (also sizes the clock pre-load identically on every rank: each
    # rank must run exactly the same number of ring steps)
    run_steps(args.warmup)
    w.synchronize()
    # calibrate the step time after the warm-up (the first steps include
    # one-time costs such as the NCCL ring's setup)
    n_cal = 20
    tw = time.perf_counter()
    run_steps(n_cal, args.warmup)
    w.synchronize()
    step_s = (time.perf_counter() - tw) / n_cal
    if dist is not None:
        t = torch.tensor([step_s], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        step_s = float(t.item())
    n_pre = int(min(5000, max(0, args.preload / max(step_s, 1e-5))))
    w.collect()
    w._metrics.clear()

    # clocks: sample while a ~1 s untimed pre-load runs, then the timed steps
    sampler = ClockSampler(_gpu_index(local_rank))
    sampler.start()
    s = args.warmup + n_cal
    for _ in range(0, n_pre, 10):
        run_steps(10, s)
        s += 10
        w.synchronize()
    w.collect()
    w._metrics.clear()

    # N=1: the timed region is K back-to-back launches of the fused step
    # kernel and nothing else, so its average launch duration is the region
    # time / K (no per-launch event pairs: each costs ~10 us of GPU time).
    # N>1: sample the bulk kernel with event pairs on ~4 of the K steps.
    if world == 1:
        w.timing = "off"
    else:
        w.timing_every = max(4, args.steps // 4)
    w._count = 0
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(w.stream)
    th0 = time.perf_counter()
    run_steps(args.steps, s)
    host_ms = (time.perf_counter() - th0) * 1e3 / args.steps
    e1.record(w.stream)
    torch.cuda.synchronize()
    barrier()
    clocks = sampler.stop()
    ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    metrics = w.metrics
    pair = w.pairable()
    launches = args.steps // 2 + args.steps % 2 if pair else args.steps
    # N=1: the region holds only the step launches: per-launch time = region
    # / launches (a two-step launch counts as two steps' worth)
    # N>1: t_bulk of a sampled launch (a pair launch reports half its time
    # per step: twice that is the launch)
    bulk_ms = ([ms * (2.0 if pair else 1.0) / args.steps] if world == 1 else
               [m["t_bulk"] * 1e3 * (2.0 if pair else 1.0) for m in metrics
                if m["t_bulk"] == m["t_bulk"]])
    sites = Lx * Ly
    mlups = sites * args.steps / (ms * 1e-3) / 1e6
    flops_step = FLOP_SITE * sites + FLOP_WALL_SITE * 6 * Lx
    gflops = flops_step * args.steps / (ms * 1e-3) / 1e9

    # dominant kernel: the fused step over the (bulk) region of this rank
    h = 3
    ey = (2 * h if grid[1] > 1 else 0)    # rows of exchanged Y edges (2-D), approx.
    kern_sites = (Lx_tile if world == 1 or pair else Lx_tile - 2 * h) * (Ly_tile - ey)
    kern_ms = float(np.mean(bulk_ms))
    achieved = BYTES_SITE * kern_sites / (kern_ms * 1e-3) / 1e9
    pk = peaks()
    hbm_peak = pk.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    if hbm_peak is None:
        hbm_peak, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"

    # the other arithmetic, same workload, same timing (every rank: the ring
    # needs the same number of steps everywhere)
    other = None
    if args.compare:
        oth = "exact" if args.arith == "fast" else "fast"
        keep = w.tparams
        w.tparams = _lib.params(tl.PhysicsParams(
            tau=0.8, gx=0.0, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
            arith=oth))
        s2 = s + args.steps + 1000

        def sustained(s0):
            """Same protocol as the headline: warm-up, the same ~preload of
            untimed steps (n_pre, identical on every rank), then K timed."""
            w._count = 0
            run_steps(3, s0)
            for _ in range(0, n_pre, 10):
                run_steps(10, s0 + 3)
                w.synchronize()
            w.collect()
            w._metrics.clear()
            barrier()
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(w.stream)
            run_steps(args.steps, s0 + 3)
            a1.record(w.stream)
            torch.cuda.synchronize()
            m = a0.elapsed_time(a1)
            if dist is not None:
                t = torch.tensor([m], device=dev)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                m = float(t.item())
            return m

        ms2 = sustained(s2)
        k2 = (ms2 / args.steps if world == 1 else
              float(np.nanmean([m["t_bulk"] * 1e3 for m in w.metrics])))
        w._metrics.clear()
        w.tparams = keep
        # A/B/A: the headline arithmetic again under the same protocol, so a
        # drift of the clock between the arms shows
        ms_again = sustained(s2 + args.steps + 2 * n_pre + 100)
        w._metrics.clear()
        ach2 = BYTES_SITE * kern_sites / (k2 * 1e-3) / 1e9
        other = {"arith": oth, "value": round(sites * args.steps / (ms2 * 1e-3) / 1e6, 3),
                 "ms_per_step": round(ms2 / args.steps, 5),
                 "gflops_fp64": round(flops_step * args.steps / (ms2 * 1e-3) / 1e9, 2),
                 "kernel_ms": round(k2, 5), "kernel_GBps": round(ach2, 1),
                 "kernel_frac_of_hbm_peak": round(ach2 / hbm_peak, 4),
                 "protocol": "A/B/A: each arm after the same %d untimed pre-load steps; "
                             "headline arithmetic re-timed after this arm" % n_pre,
                 "headline_again": {"arith": args.arith, "ms_per_step":
                                    round(ms_again / args.steps, 5),
                                    "value": round(sites * args.steps / (ms_again * 1e-3) / 1e6,
                                                   3)},
                 "parity": ("bitwise = reference" if oth == "exact"
                            else "<=1e-12 relative (tests/test_gpu_parity.py)")}

    w.timing = "sampled"
    kname = ("k_tb2<%d, 64, 2, 2, 0>" % (1 if args.arith == "exact" else 0) if pair and world == 1
             else "k_tb2<%d, 64, 2, 2, 1>" % (1 if args.arith == "exact" else 0) if pair else
             "k_site<3, %d, 4, 0, 4>" % (1 if args.arith == "exact" else 0) if world == 1 else
             "k_peer_step<%d, 0>" % (1 if args.arith == "exact" else 0))
    traffic, traffic_src = ncu_traffic(kname, args.layout)
    # the committed captures are of the configs[1] tile (1920x2048 per GPU):
    # another tile size gets the capture's bytes per site, not a per-launch
    # figure of a different launch
    traffic_site = None
    if traffic is not None:
        traffic_site = round(traffic * 1e9 / (TILE_LX * TILE_LY), 1)
        if (Lx_tile, Ly_tile) != (TILE_LX, TILE_LY):
            traffic = None
            traffic_src += ("; captured on the %dx%d tile: only its bytes per site apply"
                            % (TILE_LX, TILE_LY))
    out = None
    if rank == 0:
        lib = _lib.load()
        import ctypes
        fp = ctypes.c_double(0.0)
        if args.probe:
            _lib.check(lib.tlb_bench_dfma(200000, ctypes.byref(fp), _lib.stream_ptr()), "dfma")
        fp64_peak = fp.value / 1e12 if args.probe else float("nan")
        steps_per_launch = 2 if pair else 1
        kern_tflops = (steps_per_launch * FLOP_SITE * kern_sites) / (kern_ms * 1e-3) / 1e12
        # nominal FP64 peak at the measured SM clock: 148 SMs x 64 DFMA/clk x 2
        sm_mhz = (clocks or {}).get("sm_mhz") or 1965.0
        nominal_tf = 148 * 64 * 2 * sm_mhz * 1e6 / 1e12
        split = split_kernels(w, tl, _lib, field_desc, torch) if args.split else None
        out = {
            "metric": METRIC, "value": round(mlups, 3), "unit": "MLUPS",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms / args.steps, 5), "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (Rayleigh-Taylor initial state, reference init.py:45-64)",
            "config": {"workload": f"D2Q37 RT {Lx}x{Ly}" + (
                f" ({'1-D X' if grid[1] == 1 else f'{grid[0]}x{grid[1]}'} tiles of "
                f"{Lx_tile}x{Ly_tile}, " + ("halo exchange fused into the step kernel as "
                                            "NVLink peer stores)" if w.exchange_mode == "p2p"
                                            else "overlapped NCCL halo exchange)")
                if world > 1 else
                (" on 1 B200 (BASELINE configs[3], strong-scaling base)" if args.strong
                 else " on 1 B200 (BASELINE configs[1])")),
                "Lx": Lx, "Ly": Ly, "tiling": args.tiling, "schedule": args.schedule,
                "arith": args.arith, "layout": args.layout, "tau": 0.8, "gy": -1e-5,
                "exchange": w.exchange_mode if world > 1 else None,
                "l2": "no flush: 2 x %.2f GB state per GPU >> 126 MB L2" % (
                    37 * (Lx_tile + 6) * (Ly_tile + 6) * 8 / 1e9)},
            "gflops_fp64": round(gflops, 2),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak,
                         "unit": "GB/s", "frac": round(achieved / hbm_peak, 4),
                         "traffic": traffic, "traffic_unit": "GB per launch (ncu dram read+write)",
                         "traffic_source": traffic_src,
                         "traffic_B_per_site": traffic_site,
                         "algorithmic_bytes_per_launch_GB": round(BYTES_SITE * kern_sites / 1e9, 4),
                         "kernel": (kname + " (TWO steps per launch: propagate+bc+collide "
                                    "twice, the intermediate state in shared memory)") if pair
                         else kname + " (propagate+bc+collide)",
                         "steps_per_launch": steps_per_launch,
                         "bytes_per_site": BYTES_SITE,
                         "bytes_per_site_update": BYTES_SITE // steps_per_launch,
                         # the rate as the bandwidth a one-step kernel would need
                         # (592 B per site update): > peak means past the
                         # single-step HBM roofline
                         "single_step_equivalent_GBps": round(
                             achieved * steps_per_launch, 1),
                         "single_step_equivalent_frac": round(
                             achieved * steps_per_launch / hbm_peak, 4),
                         "sites_per_launch": kern_sites,
                         "avg_launch_ms": round(kern_ms, 5), "peak_source": peak_src,
                         "launch_timing": ("CUDA events around the K timed steps / launches "
                                           "(only step launches in the region)" if world == 1
                                           else "CUDA event pairs on sampled steps, bulk kernel"),
                         "fp64": {"achieved_tflops": round(kern_tflops, 3),
                                  "flops_per_site_update": FLOP_SITE,
                                  "count": "algorithmic (reference expression tree)",
                                  "peak_tflops_nominal_at_clock": round(nominal_tf, 3),
                                  "frac_nominal": round(kern_tflops / nominal_tf, 4),
                                  "peak_tflops_measured_dfma": round(fp64_peak, 3),
                                  "frac": round(kern_tflops / fp64_peak, 4)}},
            "clocks": clocks,
            "energy": ({"uJ_per_site_update": round(clocks["power_w_median"] * world /
                                                    (mlups * 1e6) * 1e6, 5),
                        "basis": "median nvidia-smi power.draw of rank 0's GPU during the "
                                 "pre-load + timed steps x n_gpus / MLUPS (paper Table 3 "
                                 "reports TDP-based uJ/site)"}
                       if clocks and clocks.get("power_w_median") else None),
            "host_enqueue_ms_per_step": round(host_ms, 4),
            # our kernels in the region, per rank: one per step pair (or
            # step) -- the p2p halo stores are fused in; the NCCL ring adds
            # pack, unpack and the border launch per step (+ NCCL's own)
            "gpu_launches": (launches if world == 1 or w.exchange_mode == "p2p" else
                             args.steps * 4),
        }
        if split:
            out["split"] = split
        out["parity"] = ("bitwise = reference (exact IEEE op order)" if args.arith == "exact"
                         else "fast FMA arithmetic: f, rho, T within 1e-12 relative, |du| <= "
                              "1e-12 cs after 100 RT steps (tests/test_gpu_parity.py)")
        if other:
            out["other_arith"] = other
    # e2e through the public API with host buffers
    e2e = (e2e_run(args, w, tl, torch, dist, local_rank, Lx_tile, Ly_tile, run_steps,
                   ms / args.steps) if args.e2e else None)
    if rank == 0:
        out["e2e"] = e2e
        if world == 1 and args.cpu_seconds > 0:
            mlups_cpu, nthreads, done, _, sample = cpu_oracle_rate(args.cpu_seconds)
            out["cpu_baseline"] = {"value": round(mlups_cpu, 4), "unit": "MLUPS",
                                   "cores": nthreads, "kind": "port", "sample": sample}
        emit(out)
    if dist is not None:
        dist.destroy_process_group()
    return 0


def _gpu_index(local_rank):
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if local_rank < len(ids):
            return ids[local_rank]
    return local_rank


def pcie_gbs(torch, dev, nbytes=1 << 30):
    """Measured pinned host<->device copy bandwidth (GB/s), best of 3 each way."""
    h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
    d = torch.empty(nbytes // 8, dtype=torch.float64, device=dev)
    out = {}
    for name, (dst, src) in (("h2d", (d, h)), ("d2h", (h, d))):
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dst.copy_(src, non_blocking=True)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name] = nbytes / (best * 1e-3) / 1e9
    del h, d
    return out


def e2e_run(args, w, tl, torch, dist, local_rank, Lx_tile, Ly, run_steps=None,
            device_ms_per_step=None):
    """K steps end to end through the public API with host buffers.

    Headline (`value`): what `run()` does (sim.py): the initial macroscopic
    fields (rho, ux, uy, T) in pinned host memory -> HBM -> device
    equilibrium -> K steps (RankWorker.step) -> the final populations and the
    per-step metrics back to the host (RunResult.populations / metrics).
    `populations_in`: the same with the full (Q, Lx, Ly) initial state
    uploaded instead (run(cfg, f0=...)).  Wall clock, max over ranks."""
    vs = w.vs
    state = w.physical_block()
    macro_dev = tl.moments(state.reshape(vs.Q, -1), vs)
    macro = [torch.empty((Lx_tile, Ly), dtype=torch.float64, pin_memory=True)
             for _ in range(4)]
    for h, d in zip(macro, macro_dev):
        h.copy_(d.reshape(Lx_tile, Ly).cpu())
    host_in = torch.empty((vs.Q, Lx_tile, Ly), dtype=torch.float64, pin_memory=True)
    host_in.copy_(state.cpu())
    host_out = torch.empty_like(host_in, pin_memory=True)
    world = dist.get_world_size() if dist is not None else 1

    def timed(src_macro, s0, steps=None):
        steps = args.steps if steps is None else steps
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier(device_ids=[local_rank])
        t0 = time.perf_counter()
        if src_macro:
            ts = [m.to(w.device, non_blocking=True) for m in macro]
            w.load_block(tl.equilibrium(*ts, vs))
        else:
            w.load_block(host_in)
        if run_steps is not None:
            run_steps(steps, s0)
        else:
            for s in range(steps):
                w.step(s0 + s)
        with torch.cuda.stream(w.stream):
            host_out.copy_(w.physical_block(), non_blocking=True)
        negatives = [m["negatives"] for m in w.metrics]  # D2H of per-step results
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], device=w.device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        return Lx_tile * Ly * world * steps / el / 1e6, negatives

    pops_bytes = host_in.numel() * 8 * world
    macro_bytes = 4 * Lx_tile * Ly * 8 * world
    metric_bytes = 8 * world * args.steps
    # untimed warm-up of both paths (one step each): the device temporaries
    # (upload staging, equilibrium output, result block) come from torch's
    # caching allocator afterwards instead of fresh cudaMalloc calls
    timed(False, 9_000_000, steps=1)
    timed(True, 9_500_000, steps=1)
    w.collect()
    v_pop, _ = timed(False, 10_000_000)
    v_mac, negatives = timed(True, 20_000_000)
    bw = pcie_gbs(torch, w.device)
    roof = None
    if device_ms_per_step:
        # the e2e bound: K device steps + the declared copies at the measured
        # PCIe rates (per rank; every rank copies its own tile)
        per = 1.0 / world
        ideal_s = (args.steps * device_ms_per_step * 1e-3 +
                   macro_bytes * per / (bw["h2d"] * 1e9) +
                   (pops_bytes + metric_bytes) * per / (bw["d2h"] * 1e9))
        ideal = Lx_tile * Ly * world * args.steps / ideal_s / 1e6
        roof = {"bound": "pcie + device steps", "pcie_h2d_gbs": round(bw["h2d"], 1),
                "pcie_d2h_gbs": round(bw["d2h"], 1), "ideal_mlups": round(ideal, 1),
                "frac": round(v_mac / ideal, 4),
                "note": "ideal = K x device ms/step + declared H2D/D2H bytes at the measured "
                        "pinned copy bandwidth; at K=%d the %.2f GB final-state D2H dominates"
                        % (args.steps, pops_bytes * per / 1e9)}
    return {"value": round(v_mac, 3), "unit": "MLUPS",
            "h2d_bytes_per_step": int(macro_bytes / args.steps),
            "d2h_bytes_per_step": int((pops_bytes + metric_bytes) / args.steps),
            "roofline": roof,
            "note": "as run(): pinned host (rho,ux,uy,T) -> HBM -> device equilibrium, K steps "
                    "through RankWorker (two steps per launch on one tile), final populations "
                    "+ per-step negatives -> host; wall clock, max over ranks",
            "populations_in": {"value": round(v_pop, 3), "unit": "MLUPS",
                               "h2d_bytes_per_step": int(pops_bytes / args.steps),
                               "d2h_bytes_per_step": int((pops_bytes + metric_bytes)
                                                         / args.steps),
                               "note": "as run(cfg, f0=...): the full initial state uploaded"},
            "negatives_last": int(negatives[-1]) if negatives else None}


def split_kernels(w, tl, _lib, field_desc, torch):
    """configs[1]: propagate / bc / collide timed separately (and fused), CUDA
    events on the launching stream, 5 reps each, on this rank's tile."""
    lib = _lib.load()
    g = w.geom
    full = _lib.region(g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly)
    st = w._status_ring[0].data_ptr()
    sp = w.stream.cuda_stream
    prv, nxt = field_desc(w.prv), field_desc(w.nxt)
    tp = w.tparams
    flags_fused = (_lib.F_WALL_BOT | _lib.F_WALL_TOP | _lib.F_CLAMP_Y | _lib.F_WRAP_X)
    ops = {
        "propagate": lambda: lib.tlb_propagate(prv, nxt, full, sp),
        "bc": lambda: lib.tlb_bc(nxt, tp, 1, 1, g.Hx, g.Hx + g.Lx, st, sp),
        "collide": lambda: lib.tlb_collide(nxt, nxt, full, tp, 0, st, sp),
        "fused": lambda: lib.tlb_fused(prv, nxt, full, tp, flags_fused, st, sp),
        # two whole steps per launch (temporal blocking): per-step figures below
        "two_step": lambda: lib.tlb_step2_self(prv, nxt, tp, 1, 0, 0, st, st2, 0, sp),
    }
    st2 = w._status_ring[1].data_ptr()
    res = {}
    sites = g.Lx * g.Ly
    for name, fn in ops.items():
        ts = []
        for _ in range(6):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(w.stream)
            _lib.check(fn(), name)
            b.record(w.stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        msv = float(np.median(ts[1:]))
        r = {"ms": round(msv, 4)}
        if name == "two_step":      # per step of the pair; 296 B/site per step
            r = {"ms_per_launch": round(msv, 4), "ms": round(msv / 2, 4),
                 "GBps": round(BYTES_SITE * sites / (msv * 1e-3) / 1e9, 1),
                 "mlups": round(2 * sites / (msv * 1e-3) / 1e6, 1),
                 "gflops": round(2 * FLOP_SITE * sites / (msv * 1e-3) / 1e9, 1)}
            res[name] = r
            continue
        if name == "bc":
            r["gflops"] = round(FLOP_WALL_SITE * 6 * g.Lx / (msv * 1e-3) / 1e9, 1)
            r["GBps"] = round(BYTES_SITE * 6 * g.Lx / (msv * 1e-3) / 1e9, 1)
        else:
            r["GBps"] = round(BYTES_SITE * sites / (msv * 1e-3) / 1e9, 1)
            r["mlups"] = round(sites / (msv * 1e-3) / 1e6, 1)
            if name in ("collide", "fused", "two_step"):
                r["gflops"] = round(FLOP_SITE * sites / (msv * 1e-3) / 1e9, 1)
        res[name] = r
    w.collect(raise_errors=False)
    w._metrics.clear()
    res["arith"] = "exact" if tp.arith == _lib.ARITH["exact"] else "fast"
    return res


_RESULT_OUT = None


def _reserve_stdout():
    """Keep the process's stdout for the one JSON result line: native
    libraries (NCCL's version banner, ...) and any stray print go to stderr."""
    global _RESULT_OUT
    if _RESULT_OUT is None:
        sys.stdout.flush()
        _RESULT_OUT = os.fdopen(os.dup(1), "w")
        os.dup2(2, 1)


def emit(obj):
    out = _RESULT_OUT if _RESULT_OUT is not None else sys.stdout
    print(json.dumps(obj), file=out, flush=True)


def main():
    _reserve_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arith", default="fast", choices=["exact", "fast"],
                    help="fast (default; the north star's 1e-12 contract) or exact (bitwise). "
                         "Equal speed in short bursts; under the sustained 1 kW power cap "
                         "the FP64-heavier exact arithmetic clocks lower")
    ap.add_argument("--no-compare", dest="compare", action="store_false",
                    help="skip timing the other arithmetic")
    ap.add_argument("--schedule", default="overlapped", choices=["overlapped", "staged"])
    ap.add_argument("--layout", default="column", choices=["column", "soa", "aos"],
                    help="population storage order (results are identical)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "nccl", "p2p"],
                    help="N>1 X-halo transport: NCCL ring, or NVLink peer stores fused "
                         "into the step kernel")
    ap.add_argument("--Lx", type=int, default=TILE_LX, help="tile Lx per GPU")
    ap.add_argument("--Ly", type=int, default=TILE_LY)
    ap.add_argument("--tb2-order", type=int, default=-1,
                    help="two-step kernel work order (TLB_TUNE_TB2_ORDER: -1 auto, 0, 1)")
    ap.add_argument("--tiling", default="1d",
                    help="'1d' (north star) or a rank grid 'NXxNY', e.g. 2x2 (paper's 2-D tiling)")
    ap.add_argument("--strong", action="store_true",
                    help="configs[3]: 8192x16384 total, split over the GPUs (strong scaling)")
    ap.add_argument("--preload", type=float, default=2.0, help="s of untimed load for clocks")
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-e2e", dest="e2e", action="store_false")
    ap.add_argument("--no-numpy-ref", dest="numpy_ref", action="store_false",
                    help="--impl reference: skip timing the numpy reference package itself")
    ap.add_argument("--no-split", dest="split", action="store_false")
    ap.add_argument("--no-probe", dest="probe", action="store_false",
                    help="skip the FP64 DFMA peak probe")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and world > 1:
        print(f"warning: WORLD_SIZE={world} != --gpus {args.gpus}", file=sys.stderr)
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    return gpu_arm(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
