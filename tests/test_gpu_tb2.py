"""Two steps per launch (temporal blocking, csrc/tb2.cu) against the C oracle
and against two single-step launches.

Bar: exact arithmetic bitwise (populations, per-step negative
counts, per-step failure flags); fast within 1e-12 relative.  Shapes cover
one strip and several, ragged strips, runs that cross strip boundaries,
the 8x8 minimum, walls (the materialised wall extension of the intermediate
state, runtime.py:296-305) and periodic Y.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib  # noqa: E402
from paper_1703_00185_b200.kernels import field_desc  # noqa: E402


def _setup(Lx, Ly, init, periodic, layout="column", seed=3):
    vs = tl.build_velocity_set("D2Q37")
    _lib.ensure_stencil(vs, 0)
    g = tl.LatticeGeometry(Lx, Ly, 3, 3, 37, layout)
    prv, nxt = tl.allocate_field(g, vs)
    if init == "rt":
        macro = tl.init.rayleigh_taylor_macro(Lx, Ly, vs)
    else:
        macro = tl.init.initial_macro("random", Lx, Ly, vs, seed=seed)
    f0 = tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(a), device="cuda")
                          for a in macro], vs)
    prv.pops[:, g.phys_x, g.phys_y] = f0
    return vs, g, prv, nxt, f0.cpu().numpy()


def _params(vs, arith):
    return tl.PhysicsParams(tau=0.7, gx=3e-6, gy=-2e-5, Twall_top=0.92 * vs.cs2,
                            Twall_bot=1.08 * vs.cs2, arith=arith)


def _run2(vs, g, prv, nxt, p, periodic, steps, two=True):
    """steps (even) time steps; two=True: steps/2 launches of tlb_step2_self,
    else single fused steps.  Returns the final block and per-step status."""
    lib = _lib.load()
    tp = _lib.params(p, vs)
    sts = torch.zeros((steps, _lib.STATUS_BYTES), dtype=torch.uint8, device="cuda")
    a, b = prv, nxt
    s = 0
    while s < steps:
        if two and s + 1 < steps:
            _lib.check(lib.tlb_step2_self(field_desc(a), field_desc(b), tp, int(not periodic),
                                          int(periodic), 1, sts[s].data_ptr(),
                                          sts[s + 1].data_ptr(), s, _lib.stream_ptr()), "step2")
            s += 2
        else:
            _lib.check(lib.tlb_step_self(field_desc(a), field_desc(b), tp, int(not periodic),
                                         int(periodic), 1, sts[s].data_ptr(), _lib.stream_ptr()),
                       "step")
            s += 1
        a, b = b, a
    torch.cuda.synchronize()
    out = a.pops[:, g.phys_x, g.phys_y].cpu().numpy()
    stat = [_lib.TlbStatus.from_buffer_copy(bytes(r)) for r in sts.cpu().numpy()]
    return out, stat


SHAPES = [
    (256, 128, "rt", False),     # C1: two strips of 64 rows
    (48, 300, "random", False),  # three ragged strips, walls
    (40, 245, "random", True),   # periodic Y, strip boundaries
    (8, 8, "random", False),     # the minimum tile
    (8, 8, "random", True),
    (333, 17, "rt", False),      # one strip, runs over many CTAs
    (64, 122, "random", True),   # exactly one full strip
    (64, 123, "random", False),  # one more row: two strips
]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"{s[0]}x{s[1]}-{s[2]}-{s[3]}")
def test_step2_exact_bitwise_vs_oracle(orc, shape):
    Lx, Ly, init, periodic = shape
    vs, g, prv, nxt, f0 = _setup(Lx, Ly, init, periodic)
    p = _params(vs, "exact")
    steps = 6
    got, stat = _run2(vs, g, prv, nxt, p, periodic, steps)
    orc.set_stencil(vs.c, vs.w, vs.cs2)
    want, neg = orc.run(f0, steps, orc.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top,
                                               p.Twall_bot),
                        ymode="periodic" if periodic else "walls")
    assert np.array_equal(got, want)
    assert [int(s.negatives) for s in stat] == [int(v) for v in np.asarray(neg)[:steps]]
    assert all(s.flags == 0 for s in stat)


@pytest.fixture
def tb2_tuning():
    """Restores the two-step kernel's shape and run length after a test."""
    lib = _lib.load()
    saved = []
    for key in (2, 3):
        v = ctypes.c_int(0)
        _lib.check(lib.tlb_get_tuning(key, ctypes.byref(v)), "get_tuning")
        saved.append((key, v.value))
    yield lib
    for key, v in saved:
        _lib.check(lib.tlb_set_tuning(key, v), "set_tuning")


@pytest.mark.parametrize("cfg", range(9))
def test_step2_every_shape_config_bitwise(orc, tb2_tuning, cfg):
    """Every compiled two-step kernel shape (rows x columns, CTAs/SM,
    warp-specialised) and work items from 8 columns to whole strips: exact
    bitwise vs the oracle."""
    lib = tb2_tuning
    _lib.check(lib.tlb_set_tuning(2, cfg), "cfg")
    for (Lx, Ly, init, periodic), run in (((256, 128, "rt", False), 24),
                                          ((256, 128, "rt", False), 8),
                                          ((40, 245, "random", True), 9),
                                          ((40, 245, "random", True), 100000),
                                          ((96, 300, "random", False), 40)):
        _lib.check(lib.tlb_set_tuning(3, run), "run")
        vs, g, prv, nxt, f0 = _setup(Lx, Ly, init, periodic)
        p = _params(vs, "exact")
        got, stat = _run2(vs, g, prv, nxt, p, periodic, 4)
        orc.set_stencil(vs.c, vs.w, vs.cs2)
        want, neg = orc.run(f0, 4, orc.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top,
                                               p.Twall_bot),
                            ymode="periodic" if periodic else "walls")
        assert np.array_equal(got, want), (cfg, Lx, Ly)
        assert [int(s.negatives) for s in stat] == [int(v) for v in np.asarray(neg)[:4]]


SPLIT_CFGS = (7, 8)   # one site on two threads (tb2.cu k_tb2s), fast arithmetic


@pytest.mark.parametrize("cfg", SPLIT_CFGS)
@pytest.mark.parametrize("shape", SHAPES + [(96, 300, "random", False), (256, 300, "rt", False)],
                         ids=lambda s: f"{s[0]}x{s[1]}-{s[2]}-{s[3]}")
def test_step2_split_fast_vs_oracle(orc, tb2_tuning, shape, cfg):
    """The split two-step kernel (one site on a pair of warps, partial
    moments exchanged at a named barrier): fast arithmetic within 1e-12 of
    the oracle over 6 steps, per-step negatives and flags equal; short runs
    (16 columns) and whole strips."""
    lib = tb2_tuning
    _lib.check(lib.tlb_set_tuning(2, cfg), "cfg")
    Lx, Ly, init, periodic = shape
    for run in (16, 0):
        _lib.check(lib.tlb_set_tuning(3, run), "run")
        vs, g, prv, nxt, f0 = _setup(Lx, Ly, init, periodic)
        p = _params(vs, "fast")
        got, stat = _run2(vs, g, prv, nxt, p, periodic, 6)
        orc.set_stencil(vs.c, vs.w, vs.cs2)
        want, neg = orc.run(f0, 6, orc.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top,
                                               p.Twall_bot),
                            ymode="periodic" if periodic else "walls")
        assert np.max(np.abs(got - want) / np.abs(want)) < 1e-12, (shape, run)
        assert [int(s.negatives) for s in stat] == [int(v) for v in np.asarray(neg)[:6]]
        assert all(s.flags == 0 for s in stat)


@pytest.mark.parametrize("cfg", SPLIT_CFGS)
def test_step2_split_c2_vs_fused(tb2_tuning, cfg):
    """configs[1] (1920x2048): 10 split two-step launches vs 20 fused steps,
    fast arithmetic, 1e-12; negatives per step equal."""
    lib = tb2_tuning
    _lib.check(lib.tlb_set_tuning(2, cfg), "cfg")
    vs, g, prv, nxt, _ = _setup(1920, 2048, "rt", False)
    p = _params(vs, "fast")
    state = prv.data.clone()
    two, s2 = _run2(vs, g, prv, nxt, p, False, 20, two=True)
    prv.data.copy_(state)
    one, s1 = _run2(vs, g, prv, nxt, p, False, 20, two=False)
    del state
    assert np.max(np.abs(two - one) / np.abs(one)) < 1e-12
    assert [s.negatives for s in s2] == [s.negatives for s in s1]


@pytest.mark.parametrize("cfg", SPLIT_CFGS)
def test_step2_split_reports_failures(tb2_tuning, cfg):
    """A failing site is reported once, with its step, by the split kernel."""
    lib = tb2_tuning
    _lib.check(lib.tlb_set_tuning(2, cfg), "cfg")
    vs, g, prv, nxt, _ = _setup(64, 64, "random", True)
    p = _params(vs, "fast")
    prv.pops[:, g.Hx + 10, g.Hy + 20] = -1.0
    _, stat = _run2(vs, g, prv, nxt, p, True, 2)
    assert stat[0].flags & _lib.ST_DEGENERATE


@pytest.mark.parametrize("order", [0, 1])
def test_step2_work_orders_bitwise(orc, tb2_tuning, order):
    """Both work orders of the two-step kernel (strip-major, run-major; the
    default picks run-major for fields >= 16 GB): exact bitwise vs the
    oracle, short runs so the order matters."""
    lib = tb2_tuning
    old = ctypes.c_int(0)
    _lib.check(lib.tlb_get_tuning(4, ctypes.byref(old)), "get")
    try:
        _lib.check(lib.tlb_set_tuning(4, order), "order")
        _lib.check(lib.tlb_set_tuning(3, 16), "run")
        for Lx, Ly, init, periodic in ((256, 300, "rt", False), (96, 245, "random", True)):
            vs, g, prv, nxt, f0 = _setup(Lx, Ly, init, periodic)
            p = _params(vs, "exact")
            got, stat = _run2(vs, g, prv, nxt, p, periodic, 4)
            orc.set_stencil(vs.c, vs.w, vs.cs2)
            want, neg = orc.run(f0, 4, orc.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top,
                                                   p.Twall_bot),
                                ymode="periodic" if periodic else "walls")
            assert np.array_equal(got, want), (order, Lx, Ly)
    finally:
        _lib.check(lib.tlb_set_tuning(4, old.value), "order")


@pytest.mark.parametrize("layout", ["column", "soa", "aos"])
def test_step2_equals_single_steps(layout):
    """Two steps in one launch == two fused launches, bitwise, for every
    storage layout; fast within 1e-12 (the same per-site arithmetic)."""
    for arith in ("exact", "fast"):
        for periodic in (False, True):
            vs, g, prv, nxt, _ = _setup(96, 260, "random", periodic, layout)
            p = _params(vs, arith)
            state = prv.data.clone()
            two, _ = _run2(vs, g, prv, nxt, p, periodic, 4, two=True)
            prv.data.copy_(state)
            one, _ = _run2(vs, g, prv, nxt, p, periodic, 4, two=False)
            if arith == "exact":
                assert np.array_equal(two, one), (layout, periodic)
            else:
                assert np.max(np.abs(two - one) / np.abs(one)) < 1e-12


def test_step2_reports_failures_with_their_step():
    """A site driven to rho <= 0 at level 1 is reported in step s's status,
    not step s+1's (DegenerateStateError carries the step, runtime
    collect)."""
    vs, g, prv, nxt, _ = _setup(64, 64, "random", True)
    p = _params(vs, "exact")
    prv.pops[:, g.Hx + 10, g.Hy + 20] = -1.0   # the site pulls rho < 0 at step 0
    _, stat = _run2(vs, g, prv, nxt, p, True, 2)
    assert stat[0].flags & _lib.ST_DEGENERATE


@pytest.mark.parametrize("periodic", [False, True])
def test_step2_c2_fast_and_exact_vs_fused(periodic):
    """The BASELINE configs[1] lattice (1920x2048), walls and periodic Y
    (whose wrap strips the schedule runs first): 10 two-step launches equal
    20 fused steps (exact bitwise, fast 1e-12)."""
    for arith in ("exact", "fast"):
        vs, g, prv, nxt, _ = _setup(1920, 2048, "rt", periodic)
        p = _params(vs, arith)
        state = prv.data.clone()
        two, s2 = _run2(vs, g, prv, nxt, p, periodic, 20, two=True)
        prv.data.copy_(state)
        one, s1 = _run2(vs, g, prv, nxt, p, periodic, 20, two=False)
        del state
        if arith == "exact":
            assert np.array_equal(two, one)
        else:
            assert np.max(np.abs(two - one) / np.abs(one)) < 1e-12
        assert [s.negatives for s in s2] == [s.negatives for s in s1]


@pytest.mark.parametrize("periodic", [False, True])
def test_run_uses_pairs_bitwise(orc, periodic):
    """run() on one tile with temporal="on": CUDA-graph blocks of 16 pairs
    plus loose pairs and a final single step (37 steps), snapshots at odd
    steps -- populations, per-step negatives and snapshot macro fields
    bitwise equal to the oracle (exact arithmetic)."""
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gx=2e-6, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                         Twall_bot=1.1 * vs.cs2)
    Lx, Ly, steps = 96, 150, 37
    cfg = tl.SimConfig(Lx=Lx, Ly=Ly, steps=steps, params=p, init="rayleigh-taylor",
                       walls=not periodic, periodic_y=periodic, temporal="on",
                       snapshot_every=7)
    res = tl.run(cfg)
    orc.set_stencil(vs.c, vs.w, vs.cs2)
    f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(Lx, Ly, vs.cs2))
    p6 = orc.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top, p.Twall_bot)
    ym = "periodic" if periodic else "walls"
    want, neg = orc.run(f0, steps, p6, ymode=ym)
    assert np.array_equal(res.populations, want)
    assert [m["negatives"] for m in res.metrics] == [int(v) for v in neg]
    assert [s for s, _ in res.snapshots] == [7, 14, 21, 28, 35]
    for s, m in res.snapshots:
        ref, _ = orc.run(f0, s, p6, ymode=ym)
        rho, ux, uy, T = orc.moments(ref)
        assert np.array_equal(m.rho, rho) and np.array_equal(m.T, T)
        assert np.array_equal(m.ux, ux) and np.array_equal(m.uy, uy)


def test_pairing_policy():
    """"auto" pairs steps for the fast arithmetic on large tiles only (the
    two-step kernel needs ~2 waves of strip runs to win, profiles/r02_tb2.md);
    "on" pairs any tile and both arithmetics; exact stays single-step."""
    vs = tl.build_velocity_set("D2Q37")
    fast = tl.PhysicsParams(tau=0.8, Twall_top=0.6, Twall_bot=0.7, arith="fast")
    exact = tl.PhysicsParams(tau=0.8, Twall_top=0.6, Twall_bot=0.7)

    def w(Lx, Ly, p, **kw):
        return tl.RankWorker(tl.decompose(Lx, Ly, 1, "1d")[0], vs, p, tl.Fabric(1),
                             schedule="overlapped", **kw)
    assert w(1920, 2048, fast).pairable()
    assert not w(256, 128, fast).pairable()
    assert not w(1920, 2048, exact).pairable()
    assert w(256, 128, exact, temporal="on").pairable()
    assert not w(1920, 2048, fast, temporal="off").pairable()


def test_run_fast_pairs_within_contract(orc):
    """Fast arithmetic, two steps per launch through run(): f, rho and T
    within 1e-12 relative, |du| <= 1e-12 cs after 100 steps."""
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                         arith="fast")
    res = tl.run(tl.SimConfig(Lx=256, Ly=128, steps=100, params=p, init="rayleigh-taylor",
                              temporal="on"))
    orc.set_stencil(vs.c, vs.w, vs.cs2)
    f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(256, 128, vs.cs2))
    want, _ = orc.run(f0, 100, orc.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top, p.Twall_bot))
    assert np.max(np.abs(res.populations - want) / np.abs(want)) < 1e-12
    rho, ux, uy, T = orc.moments(want)
    assert np.max(np.abs(res.macro.rho - rho) / rho) < 1e-12
    assert np.max(np.abs(res.macro.T - T) / T) < 1e-12
    du = np.hypot(res.macro.ux - ux, res.macro.uy - uy)
    assert np.max(du) <= 1e-12 * np.sqrt(vs.cs2)


def test_first_pair_launch_inside_graph_capture():
    """A fresh process whose first two-step launch is captured into a CUDA
    graph (run() with temporal="on" and >= 32 steps): the launch allocates
    nothing (the work counter is set up with the stencil)."""
    import subprocess
    import sys
    code = ("import paper_1703_00185_b200 as tl\n"
            "vs = tl.build_velocity_set('D2Q37')\n"
            "p = tl.PhysicsParams(tau=0.8, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)\n"
            "r = tl.run(tl.SimConfig(Lx=64, Ly=48, steps=64, params=p, init='rayleigh-taylor',"
            " temporal='on'))\n"
            "print('ok', len(r.metrics))\n")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert "ok 64" in out.stdout


def test_fast_pairs_1000_steps_within_contract():
    """Long-run drift: the headline path (fast arithmetic, two steps per
    launch, CUDA-graph replay) against the exact arithmetic (bitwise = the
    reference, tested against the oracle elsewhere) on C2 after 1000 steps:
    f, rho, T within 1e-12 relative, |du| <= 1e-12 cs (measured: 1.6e-13,
    1.9e-14, 2.5e-14, 1.1e-14 cs; profiles/r02z_fast_drift.jsonl)."""
    vs = tl.build_velocity_set("D2Q37")
    macro = tl.init.rayleigh_taylor_macro(1920, 2048, vs)
    f0 = tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(m)).cuda() for m in macro], vs)
    tile = tl.decompose(1920, 2048, 1, "1d")[0]
    out = {}
    for arith in ("fast", "exact"):
        p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2,
                             arith=arith)
        w = tl.RankWorker(tile, vs, p, tl.Fabric(1), schedule="overlapped", layout="column")
        assert w.pairable() == (arith == "fast")
        w.load_block(f0)
        w.run_steps(0, 1000)
        w.collect()
        out[arith] = w.physical_block()
        w.close()
    fa, fb = out["fast"], out["exact"]
    assert float(((fa - fb).abs() / fb.abs()).max()) < 1e-12
    ma, mb = tl.moments(fa.reshape(37, -1), vs), tl.moments(fb.reshape(37, -1), vs)
    assert float(((ma[0] - mb[0]).abs() / mb[0]).max()) < 1e-12
    assert float(((ma[3] - mb[3]).abs() / mb[3]).max()) < 1e-12
    assert float(torch.hypot(ma[1] - mb[1], ma[2] - mb[2]).max()) <= 1e-12 * float(np.sqrt(vs.cs2))
