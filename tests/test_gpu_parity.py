"""CUDA path vs the oracle / the reference's golden fixtures (B200 only).

Bar: bitwise equality for the exact arithmetic (every kernel and whole runs),
1e-12 relative (|du| <= 1e-12*cs for velocity) for "fast".
All compute goes through libtlb.so (the C ABI of include/tlb.h).
"""

import hashlib

import numpy as np
import pytest

from conftest import fingerprints, golden, periodic_fill, random_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib  # noqa: E402
from paper_1703_00185_b200.velocity_set import from_arrays  # noqa: E402


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="module")
def vs(stencil):
    return from_arrays(stencil["c"], stencil["w"], float(stencil["cs2"]))


@pytest.fixture(scope="module")
def kern():
    return golden("kernels.npz")


@pytest.fixture(scope="module")
def runs():
    return golden("runs.npz")


def P(arr, **kw):
    tau, gx, gy, dt, Tt, Tb = (float(v) for v in arr)
    return tl.PhysicsParams(tau=tau, gx=gx, gy=gy, dt=dt, Twall_top=Tt, Twall_bot=Tb, **kw)


def dev_pair(vs, state, Lx, Ly):
    g = tl.LatticeGeometry(Lx, Ly, 3, 3, 37)
    prv, nxt = tl.allocate_field(g, vs)
    prv.pops.copy_(torch.as_tensor(state))
    return g, prv, nxt


def test_library_is_the_compute(vs):
    lib = _lib.load()
    assert lib.tlb_version() == 1
    assert lib.tlb_device_count() >= 1


# ------------------------------------------------------------- kernels --

def test_propagate_bitwise(vs, kern):
    g, prv, nxt = dev_pair(vs, kern["prv_0"], 16, 16)
    tl.propagate(prv, nxt, vs)
    assert np.array_equal(nxt.numpy(), kern["prop_0"])


def test_bc_bitwise(vs, kern):
    g, f, _ = dev_pair(vs, kern["prop_0"], 16, 16)
    tl.bc(f, P(kern["params"]), vs)
    assert np.array_equal(f.numpy(), kern["bc_0"])


@pytest.mark.parametrize("seed", [0, 23])
def test_collide_moments_bitwise(vs, kern, orc, seed):
    prv = kern[f"prv_{seed}"]
    nxt = np.zeros_like(prv)
    orc.propagate(prv.copy(), nxt, 3)
    blk = nxt[:, 3:19, 3:19]
    # numpy in -> numpy out (computed by the CUDA kernel)
    out = tl.collide(blk, P(kern["params"]), vs)
    assert isinstance(out, np.ndarray)
    assert np.array_equal(out, kern[f"collide_{seed}"])
    # torch strided view in -> torch out
    g, f, _ = dev_pair(vs, nxt, 16, 16)
    out_t = tl.collide(f.pops[:, 3:19, 3:19], P(kern["params"]), vs)
    assert np.array_equal(out_t.cpu().numpy(), kern[f"collide_{seed}"])
    mom = tl.moments(f.pops[:, 3:19, 3:19], vs)
    assert np.array_equal(np.stack([m.cpu().numpy() for m in mom]), kern[f"mom_{seed}"])
    sh = tl.apply_shift(*mom[1:], P(kern["params"]))
    assert np.array_equal(np.stack([s.cpu().numpy() for s in sh]), kern[f"shift_{seed}"])


def test_fused_bitwise(vs, kern):
    g, prv, nxt = dev_pair(vs, kern["prv_0"], 16, 16)
    tl.propagate_collide_fused(prv, nxt, P(kern["params"]), vs,
                               (slice(4, 17), slice(6, 16)))
    assert np.array_equal(nxt.numpy(), kern["fused_0"])


@pytest.mark.parametrize("order", [2, 3, 4])
def test_equilibrium_bitwise(vs, kern, order):
    out = tl.equilibrium(*kern["eq_in"], vs, order=order)
    assert np.array_equal(out, kern[f"eq_out_{order}"])


def test_rest_equilibrium_is_w(vs):
    # reference tests/test_kernels.py:124-126
    f = tl.equilibrium(np.float64(1.0), 0.0, 0.0, np.float64(vs.cs2), vs)
    assert np.array_equal(f, vs.w)


def test_fast_collide_close(vs, kern, orc):
    prv = kern["prv_0"]
    nxt = np.zeros_like(prv)
    orc.propagate(prv.copy(), nxt, 3)
    blk = nxt[:, 3:19, 3:19]
    out = tl.collide(blk, P(kern["params"], arith="fast"), vs)
    ref = kern["collide_0"]
    # random states are far from equilibrium, so some outputs cancel to ~0:
    # bound the error by the site's population scale
    scale = np.abs(ref).max(axis=0, keepdims=True)
    assert np.max(np.abs(out - ref) / scale) < 1e-13


# ---------------------------------------------------------- region rules --

def test_region_contract(vs):
    g = tl.LatticeGeometry(8, 8, 3, 3, 37)
    prv, nxt = tl.allocate_field(g, vs)
    with pytest.raises(tl.ContractViolation):
        tl.propagate(prv, nxt, vs, (slice(0, g.NX), g.phys_y))
    with pytest.raises(tl.ContractViolation):
        tl.propagate_collide_fused(prv, nxt, tl.PhysicsParams(tau=0.8), vs,
                                   (g.phys_x, g.phys_y), exclude_y=[(g.Hy, g.Hy + 3)])


def test_fused_empty_region_noop(vs):
    g = tl.LatticeGeometry(8, 8, 3, 3, 37)
    prv, nxt = tl.allocate_field(g, vs)
    prv.pops.copy_(torch.as_tensor(random_state(g.NX, g.NY, seed=4)))
    before = nxt.numpy().copy()
    tl.propagate_collide_fused(prv, nxt, tl.PhysicsParams(tau=0.8), vs,
                               (slice(g.Hx, g.Hx), g.phys_y))
    assert np.array_equal(nxt.numpy(), before)


def test_degenerate_state_raises(vs):
    with pytest.raises(tl.DegenerateStateError):
        tl.moments(np.zeros((37, 3)), vs)
    with pytest.raises(tl.DegenerateStateError):
        tl.collide(np.zeros((37, 2)), tl.PhysicsParams(tau=0.8), vs)


def test_shift_domain_error(vs):
    with pytest.raises(tl.DomainError):
        tl.apply_shift(0.0, 0.0, 0.5, tl.PhysicsParams(tau=10.0, gy=-0.5))
    ub, vb, Tb = tl.apply_shift(0.0, 0.0, 0.5, tl.PhysicsParams(tau=1.0, gy=-0.01))
    assert ub == 0.0 and abs(vb + 0.01) < 1e-15 and abs(Tb - (0.5 - 5e-5)) < 1e-15


def test_equilibrium_domain_error(vs):
    with pytest.raises(tl.DomainError):
        tl.equilibrium(np.float64(-1.0), 0.0, 0.0, np.float64(0.3), vs)


def test_count_negative(vs):
    f = np.ones((37, 4, 5))
    f[3, 1, 2] = -1.0
    f[30, 0, 0] = -2.0
    assert tl.count_negative(f) == 2


# ------------------------------------------------------------ whole runs --

def _run(vs, f0, steps, params, schedule, Np=1, walls=True, periodic_y=False):
    """Drive RankWorkers directly with an explicit f0 (independent of the host's
    LAPACK-derived weights), like sim.run does."""
    Q, Lx, Ly = f0.shape
    tiles = tl.decompose(Lx, Ly, Np, "1d", periodic_y=periodic_y)
    fab = tl.Fabric(Np)
    ws = []
    for t in tiles:
        w = tl.RankWorker(t, vs, params, fab, schedule=schedule, walls=walls,
                          periodic_y=periodic_y)
        w.load_block(torch.as_tensor(f0[:, t.x0:t.x0 + t.Lx]))
        ws.append(w)
    for s in range(steps):
        for phase in ("step_begin", "step_mid", "step_end"):
            for w in ws:
                getattr(w, phase)(s)
    out = np.empty_like(f0)
    negs = []
    for w in ws:
        w.synchronize()
        out[:, w.tile.x0:w.tile.x0 + w.tile.Lx] = w.physical_block().cpu().numpy()
        negs.append([m["negatives"] for m in w.metrics])
    return out, np.sum(negs, axis=0) if steps else []


@pytest.mark.parametrize("schedule", ["staged", "overlapped"])
def test_run_rt_golden(vs, runs, schedule):
    out, neg = _run(vs, runs["rt_f0"], 20, P(runs["rt_params"]), schedule)
    assert np.array_equal(out, runs["rt_f20"])
    assert np.array_equal(neg, runs["rt_f20_negatives"])


@pytest.mark.parametrize("schedule,Np", [("staged", 1), ("overlapped", 1),
                                         ("staged", 4), ("overlapped", 4),
                                         ("overlapped", 2)])
def test_run_random_walls_golden_rank_invariance(vs, runs, schedule, Np):
    out, _ = _run(vs, runs["rw_f0"], 6, P(runs["rw_params"]), schedule, Np=Np)
    assert np.array_equal(out, runs["rw_f6"])


@pytest.mark.parametrize("schedule", ["staged", "overlapped"])
def test_run_periodic_golden(vs, runs, schedule):
    out, _ = _run(vs, runs["pp_f0"], 10, P(runs["pp_params"]), schedule, walls=False,
                  periodic_y=True)
    assert np.array_equal(out, runs["pp_f10"])


@pytest.fixture(scope="module")
def rt256(vs, orc):
    f0 = tl.equilibrium(*[torch.as_tensor(a).cuda() for a in
                          tl.init.rayleigh_taylor_macro(256, 128, vs)], vs).cpu().numpy()
    return f0


def test_rt256_fingerprint(vs, runs, rt256):
    """SURVEY §8c known answer (RT 256x128, 100 steps) on the GPU."""
    fp = fingerprints()
    assert sha16(rt256) == fp["rt256_f0"]
    for schedule in ("overlapped", "staged"):
        out, _ = _run(vs, rt256, 100, P(runs["rt_params"]), schedule)
        assert sha16(out) == fp["rt256_f100"], schedule


def test_rt256_rank_invariance(vs, runs, rt256):
    one, _ = _run(vs, rt256, 30, P(runs["rt_params"]), "overlapped", Np=1)
    for Np in (2, 4, 8):
        many, _ = _run(vs, rt256, 30, P(runs["rt_params"]), "overlapped", Np=Np)
        assert np.array_equal(one, many), Np


def test_rt256_fast_within_tolerance(vs, runs, rt256, orc):
    """fast arithmetic: 1e-12 relative on f, rho, T; |du| <= 1e-12 * cs."""
    ref, _ = _run(vs, rt256, 100, P(runs["rt_params"]), "overlapped")
    got, _ = _run(vs, rt256, 100, P(runs["rt_params"], arith="fast"), "overlapped")
    assert np.max(np.abs(got - ref) / np.abs(ref)) < 1e-12
    mr = orc.moments(ref)
    mg = orc.moments(got)
    cs = np.sqrt(vs.cs2)
    assert np.max(np.abs(mg[0] - mr[0]) / mr[0]) < 1e-12
    assert np.max(np.abs(mg[3] - mr[3]) / mr[3]) < 1e-12
    du = np.hypot(mg[1] - mr[1], mg[2] - mr[2])
    assert np.max(du) <= 1e-12 * cs


def test_run_api_matches_oracle(vs, orc):
    """sim.run (the public entry) vs the oracle on identical inputs."""
    vsb = tl.build_velocity_set("D2Q37")
    orc.set_stencil(vsb.c, vsb.w, vsb.cs2)
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vsb.cs2,
                         Twall_bot=1.1 * vsb.cs2)
    for Np, schedule in ((1, "overlapped"), (2, "overlapped"), (1, "staged")):
        res = tl.run(tl.SimConfig(Lx=96, Ly=40, Np=Np, steps=7, params=p,
                                  init="rayleigh-taylor", schedule=schedule))
        f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(96, 40, vsb.cs2))
        want, neg = orc.run(f0, 7, orc.params6(0.8, 0.0, -1e-5, 1.0, p.Twall_top,
                                                 p.Twall_bot))
        assert np.array_equal(res.populations, want), (Np, schedule)
        assert res.mlups > 0
        assert len(res.metrics) == 7 * Np
        rho, ux, uy, T = orc.moments(want)
        assert np.array_equal(res.macro.rho, rho) and np.array_equal(res.macro.T, T)
    orc.set_stencil(vs.c, vs.w, vs.cs2)


@pytest.mark.parametrize("Lx,Ly", [(7, 13), (3, 6), (5, 9), (130, 7), (9, 4), (8, 5)])
def test_ragged_sizes_bitwise(vs, orc, Lx, Ly):
    rng = np.random.default_rng(Lx * 100 + Ly)
    f0 = orc.equilibrium(1.0 + 0.01 * rng.standard_normal((Lx, Ly)),
                         0.01 * rng.standard_normal((Lx, Ly)),
                         0.01 * rng.standard_normal((Lx, Ly)),
                         vs.cs2 * (1 + 0.01 * rng.standard_normal((Lx, Ly))))
    p = tl.PhysicsParams(tau=0.8, gx=1e-5, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    p6 = orc.params6(0.8, 1e-5, -1e-4, 1.0, 0.6, 0.75)
    want, _ = orc.run(f0, 5, p6)
    for schedule in ("overlapped", "staged"):
        got, _ = _run(vs, f0, 5, p, schedule)
        assert np.array_equal(got, want), schedule


def test_large_c2_two_steps_bitwise(vs, orc):
    """C2 size (1920x2048): 2 fused steps equal the oracle bit for bit."""
    Lx, Ly = 1920, 2048
    macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
    f0 = tl.equilibrium(*[torch.as_tensor(a).cuda() for a in macro], vs).cpu().numpy()
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    got, neg = _run(vs, f0, 2, p, "overlapped")
    want, wneg = orc.run(f0, 2, orc.params6(0.8, 0.0, -1e-5, 1.0, p.Twall_top, p.Twall_bot))
    assert np.array_equal(got, want)
    assert np.array_equal(neg, wneg)


def test_error_surfaces_with_step(vs):
    """A degenerate state inside the step loop is raised at collect()."""
    g = tl.LatticeGeometry(8, 8, 3, 3, 37)
    tiles = tl.decompose(8, 8, 1, "1d")
    w = tl.RankWorker(tiles[0], vs, tl.PhysicsParams(tau=0.8), tl.Fabric(1),
                      schedule="overlapped")
    w.load_block(torch.zeros((37, 8, 8), dtype=torch.float64))
    w.step(0)
    with pytest.raises(tl.DomainError):
        w.collect()


def test_rt256_1000_steps_exact_bitwise_and_fast_drift(vs, runs, rt256, orc):
    """1000 RT steps: exact stays bitwise equal to the oracle; fast stays
    within the north star's 1e-12 relative contract."""
    p6 = orc.params6(*runs["rt_params"])
    want, _ = orc.run(rt256, 1000, p6)
    got, _ = _run(vs, rt256, 1000, P(runs["rt_params"]), "overlapped")
    assert np.array_equal(got, want)
    fast, _ = _run(vs, rt256, 1000, P(runs["rt_params"], arith="fast"), "overlapped")
    rel = np.max(np.abs(fast - want) / np.abs(want))
    print("fast drift after 1000 steps:", rel)
    assert rel < 1e-12


@pytest.mark.parametrize("case", range(24))
def test_randomised_configs_bitwise(vs, orc, case):
    """Seeded random configurations through run() against the C oracle,
    bitwise: lattice shape, tau, body force, wall temperatures, walls or
    periodic Y, rank count and tiling (in-process ranks), schedule,
    storage layout, random or Rayleigh-Taylor start, 1-9 steps."""
    rng = np.random.default_rng(1000 + case)
    periodic = bool(rng.integers(2))
    tiling_choice = int(rng.integers(3))
    Np, tiling = [(1, "1d"), (2, "1d"), (4, (2, 2))][tiling_choice]
    nx, ny = (Np, 1) if tiling == "1d" else tiling
    Lx = nx * int(rng.integers(7, 40))
    Ly = ny * int(rng.integers(7, 40))
    tau = float(rng.uniform(0.55, 2.0))
    gx, gy = (float(v) for v in rng.normal(0.0, 2e-5, 2))
    Tt, Tb = (float(v) * vs.cs2 for v in rng.uniform(0.85, 1.15, 2))
    p = tl.PhysicsParams(tau=tau, gx=gx, gy=gy, Twall_top=Tt, Twall_bot=Tb)
    init = ["random", "rayleigh-taylor"][int(rng.integers(2))]
    steps = int(rng.integers(1, 10))
    res = tl.run(tl.SimConfig(
        Lx=Lx, Ly=Ly, Np=Np, tiling=tiling, steps=steps, params=p, init=init,
        init_kwargs={"seed": case} if init == "random" else {},
        walls=not periodic, periodic_y=periodic,
        schedule=["overlapped", "staged"][int(rng.integers(2))],
        layout=["column", "soa", "aos"][int(rng.integers(3))]))
    f0 = tl.init.build_initial_state(init, Lx, Ly, vs,
                                     **({"seed": case} if init == "random" else {}))
    want, _ = orc.run(f0.cpu().numpy(), steps,
                      orc.params6(tau, gx, gy, 1.0, Tt, Tb),
                      ymode="periodic" if periodic else "walls")
    assert np.array_equal(res.populations, want), (case, Lx, Ly, Np, tiling, periodic)


def _macro_contract(orc, vs, got, want):
    """SURVEY §8c on (Q, Lx, Ly) blocks: f, rho and T within 1e-12 relative,
    |du| <= 1e-12 * cs.  Returns the four worst errors."""
    rel_f = np.max(np.abs(got - want) / np.abs(want))
    mg, mw = orc.moments(got), orc.moments(want)
    rel_rho = np.max(np.abs(mg[0] - mw[0]) / mw[0])
    rel_T = np.max(np.abs(mg[3] - mw[3]) / mw[3])
    du = np.max(np.hypot(mg[1] - mw[1], mg[2] - mw[2])) / np.sqrt(vs.cs2)
    assert rel_f < 1e-12 and rel_rho < 1e-12 and rel_T < 1e-12 and du <= 1e-12, \
        (rel_f, rel_rho, rel_T, du)
    return rel_f, rel_rho, rel_T, du


def test_c2_headline_fast_20_steps_vs_oracle(vs, orc):
    """The bench's headline path at the bench config: C2 (1920x2048, RT,
    walls), fast arithmetic through RankWorker.run_steps -- the two-step
    kernel (tlb_step2_self) plus CUDA-graph replay, exactly what bench.py
    times -- for 20 steps against the C oracle on the same f0."""
    Lx, Ly, n = 1920, 2048, 20
    macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
    f0 = tl.equilibrium(*[torch.as_tensor(a).cuda() for a in macro], vs).cpu().numpy()
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                         arith="fast")
    tile = tl.decompose(Lx, Ly, 1, "1d")[0]
    w = tl.RankWorker(tile, vs, p, tl.Fabric(1), schedule="overlapped", layout="column")
    assert w.pairable()
    w.load_block(torch.as_tensor(f0))
    w.run_steps(0, n)
    got = w.physical_block().cpu().numpy()
    w.collect()
    want, _ = orc.run(f0, n, orc.params6(0.8, 0.0, -1e-5, 1.0, p.Twall_top, p.Twall_bot))
    print("C2 fast vs oracle (f, rho, T, |du|/cs):", _macro_contract(orc, vs, got, want))
