"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container (where /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is pure Python/numpy (`thermolb`), so it cannot travel to the
GPU box; these small .npz files carry its outputs instead.  Every array is
produced by calling the reference's own public functions (no re-implementation
here), so the fixtures pin both the C oracle (`oracle/`) and the CUDA path.

Fixtures (all float64 unless noted):
  stencil.npz     c (37,2) int64, w (37,), cs2, plus ex/ey/q per l exactly as
                  `kernels.equilibrium` computes them (kernels.py:87-98)
  kernels.npz     per-kernel input/output pairs on 16x16 / 12x16 tiles
                  (propagate kernels.py:168, bc :180, collide :139,
                  fused :206, moments :41, equilibrium :74, apply_shift :128)
  runs.npz        multi-step runs through `run()` (sim.py:62): RT 32x24 with
                  walls, random 16x16 with walls (Np=1 staged, Np=4 1-D
                  overlapped), periodic 16x16 conservation
  rt_init.npz     the (rho, T) macro fields `init.rayleigh_taylor` hands to
                  `equilibrium` for RT 64x32 (init.py:45-64), captured by
                  wrapping the reference's equilibrium
  halo.npz        face payloads of the reference RankWorker: pack_x(+/-1)
                  on a 1-D 2-rank tile (runtime.py:199-208) and pack_y(+/-1)
                  on a 2x2 tile (:226-235) of a random padded field, plus
                  the fields after unpack_x / unpack_y of those payloads
                  into a zeroed receiver (:210-224, :237-246)
  fingerprints.json  SHA-256 prefixes of w, f0 and f100 for RT 256x128 x 100
                  steps (the SURVEY §8c known answer), re-derived here
"""

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import thermolb  # noqa: E402
from thermolb import (LatticeGeometry, PhysicsParams, SimConfig,  # noqa: E402
                      allocate_field, apply_shift, bc, build_velocity_set,
                      collide, equilibrium, moments, propagate,
                      propagate_collide_fused, run)
import thermolb.init as ref_init  # noqa: E402

sys.path.insert(0, "/root/reference/pkg/tests")
from conftest import periodic_fill, random_state  # noqa: E402


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:16]


def main():
    vs = build_velocity_set("D2Q37")
    cs = np.sqrt(vs.cs2)
    ex = np.array([vs.c[l, 0] / cs for l in range(vs.Q)])
    ey = np.array([vs.c[l, 1] / cs for l in range(vs.Q)])
    q = ex * ex + ey * ey
    np.savez(os.path.join(HERE, "stencil.npz"), c=vs.c, w=vs.w,
             cs2=np.float64(vs.cs2), cs=np.float64(cs), ex=ex, ey=ey, q=q)

    # ---------------------------------------------------------- kernels --
    k = {}
    g = LatticeGeometry(16, 16, 3, 3, vs.Q)
    params = PhysicsParams(tau=0.8, gx=3e-6, gy=-1e-4, Twall_top=0.62,
                           Twall_bot=0.81)
    k["params"] = np.array([params.tau, params.gx, params.gy, params.dt,
                            params.Twall_top, params.Twall_bot])
    for seed in (0, 23):
        full = seed == 0  # full-field arrays for one seed keep the file small
        prv, nxt = allocate_field(g, vs)
        prv.pops[...] = random_state(g, vs, seed=seed)
        periodic_fill(prv)
        k[f"prv_{seed}"] = prv.pops.copy()
        # propagate over the full physical region (kernels.py:168-177)
        propagate(prv, nxt, vs)
        if full:
            k[f"prop_{seed}"] = nxt.pops.copy()
        # bc on the propagated field, both walls (kernels.py:180-203)
        bcf = type(nxt)(g, "nxt", nxt.pops.copy())
        bc(bcf, params, vs)
        if full:
            k[f"bc_{seed}"] = bcf.pops.copy()
        # collide on the physical block of the propagated field (:139-146)
        blk = nxt.pops[:, g.phys_x, g.phys_y]
        k[f"collide_{seed}"] = collide(blk, params, vs)
        # fused over a sub-region (kernels.py:206-224)
        fz = type(nxt)(g, "nxt")
        region = (slice(g.Hx + 1, g.Hx + 14), slice(g.Hy + 3, g.Hy + 13))
        propagate_collide_fused(prv, fz, params, vs, region)
        if full:
            k[f"fused_{seed}"] = fz.pops.copy()
        rho, ux, uy, T = moments(blk, vs)
        k[f"mom_{seed}"] = np.stack([rho, ux, uy, T])
        ub, vb, Tb = apply_shift(ux, uy, T, params)
        k[f"shift_{seed}"] = np.stack([ub, vb, Tb])
    rng = np.random.default_rng(5)
    n = 64
    rho = 0.5 + rng.random(n)
    ux = 0.1 * rng.standard_normal(n)
    uy = 0.1 * rng.standard_normal(n)
    T = vs.cs2 * (0.8 + 0.4 * rng.random(n))
    k["eq_in"] = np.stack([rho, ux, uy, T])
    for order in (2, 3, 4):
        k[f"eq_out_{order}"] = equilibrium(rho, ux, uy, T, vs, order=order)
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **k)

    # ------------------------------------------------------------- runs --
    r = {}
    p_rt = PhysicsParams(tau=0.8, gx=0.0, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                         Twall_bot=1.1 * vs.cs2)
    r["rt_params"] = np.array([p_rt.tau, p_rt.gx, p_rt.gy, p_rt.dt,
                               p_rt.Twall_top, p_rt.Twall_bot])
    cfg = dict(Lx=32, Ly=24, model="D2Q37", params=p_rt, init="rayleigh-taylor")
    r["rt_f0"] = run(SimConfig(Np=1, steps=0, **cfg)).populations
    res = run(SimConfig(Np=1, tiling="1d", schedule="staged", steps=20, **cfg))
    r["rt_f20"] = res.populations
    r["rt_f20_macro"] = np.stack([res.macro.rho, res.macro.ux, res.macro.uy,
                                  res.macro.T])
    r["rt_f20_negatives"] = np.array([m["negatives"] for m in res.metrics])
    res4 = run(SimConfig(Np=4, tiling="1d", schedule="overlapped", steps=20, **cfg))
    assert np.array_equal(res4.populations, res.populations)

    p_w = PhysicsParams(tau=0.8, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    r["rw_params"] = np.array([p_w.tau, p_w.gx, p_w.gy, p_w.dt,
                               p_w.Twall_top, p_w.Twall_bot])
    kw = dict(Lx=16, Ly=16, model="D2Q37", params=p_w, init="random",
              init_kwargs={"seed": 5})
    r["rw_f0"] = run(SimConfig(Np=1, steps=0, **kw)).populations
    one = run(SimConfig(Np=1, tiling="1d", schedule="staged", steps=6, **kw))
    four = run(SimConfig(Np=4, tiling="1d", schedule="overlapped", steps=6, **kw))
    assert np.array_equal(one.populations, four.populations)
    r["rw_f6"] = one.populations

    p_p = PhysicsParams(tau=0.8)
    r["pp_params"] = np.array([p_p.tau, p_p.gx, p_p.gy, p_p.dt,
                               p_p.Twall_top, p_p.Twall_bot])
    kwp = dict(Lx=16, Ly=16, model="D2Q37", params=p_p, walls=False,
               periodic_y=True, init="random", init_kwargs={"seed": 7})
    r["pp_f0"] = run(SimConfig(Np=1, tiling=(1, 1), steps=0, **kwp)).populations
    r["pp_f10"] = run(SimConfig(Np=1, tiling=(1, 1), schedule="staged",
                                steps=10, **kwp)).populations
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **r)

    # ---------------------------------------------------------- RT init --
    captured = {}
    orig = ref_init.equilibrium

    def spy(rho, ux, uy, T, vs_, *a, **kw_):
        captured.update(rho=np.array(rho), ux=np.array(ux), uy=np.array(uy),
                        T=np.array(T))
        return orig(rho, ux, uy, T, vs_, *a, **kw_)

    ref_init.equilibrium = spy
    try:
        f0 = ref_init.rayleigh_taylor(64, 32, vs)
    finally:
        ref_init.equilibrium = orig
    np.savez(os.path.join(HERE, "rt_init.npz"), rho=captured["rho"],
             T=captured["T"], f0_sha=np.array(sha16(f0)))
    captured.clear()
    ref_init.equilibrium = spy
    try:
        ref_init.random_near_equilibrium(16, 16, vs, seed=7)
    finally:
        ref_init.equilibrium = orig
    np.savez(os.path.join(HERE, "random_init.npz"), **captured)

    # ------------------------------------------------------------- io --
    import tempfile
    import thermolb.io as ref_io
    T = r["rt_f20_macro"][3]
    with tempfile.TemporaryDirectory() as td:
        ref_io.write_pgm(os.path.join(td, "t.pgm"), T)
        pgm = open(os.path.join(td, "t.pgm"), "rb").read()
        from thermolb.geometry import MacroFields
        mf = MacroFields(*r["rt_f20_macro"][:, :4, :3])
        ref_io.write_macro_csv(os.path.join(td, "m.csv"), mf)
        csv_txt = open(os.path.join(td, "m.csv")).read()
    np.savez(os.path.join(HERE, "io.npz"), T=T, pgm=np.frombuffer(pgm, dtype=np.uint8),
             macro_small=r["rt_f20_macro"][:, :4, :3], csv=np.array(csv_txt))

    # ---------------------------------------------------------- D2Q9 --
    v9 = build_velocity_set("D2Q9")
    g9 = LatticeGeometry(8, 8, 3, 3, 9)
    d9 = {}
    prv, nxt = allocate_field(g9, v9)
    prv.pops[...] = random_state(g9, v9, seed=29)
    periodic_fill(prv)
    d9["prv"] = prv.pops.copy()
    propagate(prv, nxt, v9)
    d9["prop"] = nxt.pops.copy()
    p9 = PhysicsParams(tau=0.8, gx=2e-5, gy=-1e-4, Twall_top=0.3, Twall_bot=0.36)
    d9["params"] = np.array([p9.tau, p9.gx, p9.gy, p9.dt, p9.Twall_top, p9.Twall_bot])
    b9 = type(nxt)(g9, "nxt", nxt.pops.copy())
    bc(b9, p9, v9)
    d9["bc"] = b9.pops.copy()
    d9["collide"] = collide(nxt.pops[:, g9.phys_x, g9.phys_y], p9, v9)
    fz = type(nxt)(g9, "nxt")
    propagate_collide_fused(prv, fz, p9, v9, (slice(4, 10), slice(5, 9)))
    d9["fused"] = fz.pops.copy()
    kw9 = dict(Lx=16, Ly=12, model="D2Q9", params=p9, init="random", init_kwargs={"seed": 4})
    d9["run_f0"] = run(SimConfig(Np=1, steps=0, **kw9)).populations
    one9 = run(SimConfig(Np=1, schedule="staged", steps=10, **kw9))
    two9 = run(SimConfig(Np=2, tiling="1d", schedule="overlapped", steps=10, **kw9))
    assert np.array_equal(one9.populations, two9.populations)
    d9["run_f10"] = one9.populations
    np.savez_compressed(os.path.join(HERE, "d2q9.npz"), **d9)

    # -------------------------------------------------------- planner --
    from thermolb import planner as P
    rng = np.random.default_rng(0)
    rows, ins = [], []
    tab = P.BandwidthTable([1e3, 1e5, 1e7], [2e9, 3e10, 6e11])
    for k in range(40):
        Lx = int(rng.integers(64, 4000)); Ly = Lx if k % 4 == 0 else int(rng.integers(64, 4000))
        Np = int(rng.integers(1, 64))
        Bx = float(rng.uniform(1e8, 1e12)); By = float(rng.uniform(1e8, 1e12))
        beta = float(rng.uniform(1e-10, 1e-7)); S = float(rng.uniform(8, 400))
        use_tab = k % 3 == 0
        inp = P.CostModelInput(Lx, Ly, Np, tab if use_tab else Bx, tab if use_tab else By,
                               beta, S)
        real, best = P.optimal_grid(inp)
        vals = [P.predict_1d(inp).T_total, P.predict_2d(inp).T_total,
                P.predict_2d(inp, grid=best).T_total, P.predict_1d_overlap(inp).T_total,
                P.predict_1d_overlap(inp).scale_violation,
                P.predict_2d_overlap(inp).T_total if Lx == Ly else np.nan,
                P.comm_time_2d(inp, *best), real[0], real[1], best[0], best[1],
                P.surface_over_volume(Np, 2), P.brent_bound(beta, Lx * Ly, Np)]
        ins.append([Lx, Ly, Np, Bx, By, beta, S, use_tab])
        rows.append(vals)
    np.savez(os.path.join(HERE, "planner.npz"), inputs=np.array(ins, dtype=np.float64),
             outputs=np.array(rows, dtype=np.float64), tab_sizes=tab.sizes, tab_bw=tab.bandwidths)

    # ---------------------------------------------------- fingerprints --
    fp = {"w": sha16(vs.w), "cs2": float.hex(float(vs.cs2))}
    cfg = SimConfig(Lx=256, Ly=128, model="D2Q37", Np=1, tiling="1d",
                    schedule="staged", steps=100, params=p_rt,
                    init="rayleigh-taylor")
    f0 = run(SimConfig(**{**cfg.__dict__, "steps": 0})).populations
    fp["rt256_f0"] = sha16(f0)
    fp["rt256_f0_sum"] = float(f0.sum())
    res = run(cfg)
    fp["rt256_f100"] = sha16(res.populations)
    fp["rt256_f100_sum"] = float(res.populations.sum())
    fp["rt256_negatives"] = [m["negatives"] for m in res.metrics][:5]
    fp["generated_with"] = {"numpy": np.__version__,
                            "thermolb": thermolb.__version__}
    with open(os.path.join(HERE, "fingerprints.json"), "w") as fh:
        json.dump(fp, fh, indent=1)
    print(json.dumps(fp, indent=1))
    halo()


def halo():
    """halo.npz: the reference's own face payload byte order."""
    from thermolb.runtime import Fabric, RankWorker, decompose
    vs = build_velocity_set("D2Q37")
    p = PhysicsParams(tau=0.8, Twall_top=0.6, Twall_bot=0.8)
    h = {}
    for tag, Lx, Ly, Np, tiling in (("x", 14, 10, 2, "1d"), ("y", 14, 10, 4, (2, 2))):
        tiles = decompose(Lx, Ly, Np, tiling, periodic_y=tag == "y")
        w = RankWorker(tiles[0], vs, p, Fabric(Np))
        rx = RankWorker(tiles[0], vs, p, Fabric(Np))
        g = w.geom
        w.prv.pops[...] = random_state(g, vs, seed=21 if tag == "x" else 22)
        h[f"{tag}_field"] = w.prv.pops.copy()
        h[f"{tag}_shape"] = np.array([tiles[0].Lx, tiles[0].Ly])
        for sign in (1, -1):
            pay = (w.pack_x if tag == "x" else w.pack_y)(w.prv, sign).copy()
            h[f"{tag}_pack{'+' if sign == 1 else '-'}"] = pay
            rx.prv.pops[...] = 0.0
            (rx.unpack_x if tag == "x" else rx.unpack_y)(rx.prv, sign, pay)
            h[f"{tag}_unpack{'+' if sign == 1 else '-'}"] = rx.prv.pops.copy()
    np.savez_compressed(os.path.join(HERE, "halo.npz"), **h)


if __name__ == "__main__":
    if sys.argv[1:] == ["halo"]:
        halo()
    else:
        main()
