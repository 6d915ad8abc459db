"""D2Q9 (and any non-specialised stencil) through the generic kernels, and
the generic path cross-checked against the specialised D2Q37 kernels.

Mirrors the reference's D2Q9 tests (tests/test_kernels.py:23-33, 140-151,
192-197, 264-269, 302-321; test_runtime.py:58-61, 137-158) and compares
with D2Q9 fixtures produced by the reference (tests/golden/d2q9.npz).
"""

import numpy as np
import pytest

from conftest import golden, random_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib  # noqa: E402


@pytest.fixture(scope="module")
def d2q9():
    return tl.build_velocity_set("D2Q9")


@pytest.fixture(scope="module")
def g9():
    return golden("d2q9.npz")


def P(arr, **kw):
    tau, gx, gy, dt, Tt, Tb = (float(v) for v in arr)
    return tl.PhysicsParams(tau=tau, gx=gx, gy=gy, dt=dt, Twall_top=Tt, Twall_bot=Tb, **kw)


def field(vs, state, Lx, Ly):
    g = tl.LatticeGeometry(Lx, Ly, 3, 3, vs.Q)
    prv, nxt = tl.allocate_field(g, vs)
    if state is not None:
        prv.pops.copy_(torch.as_tensor(state))
    return g, prv, nxt


def test_d2q9_kernels_bitwise(d2q9, g9):
    p = P(g9["params"])
    g, prv, nxt = field(d2q9, g9["prv"], 8, 8)
    tl.propagate(prv, nxt, d2q9)
    assert np.array_equal(nxt.numpy(), g9["prop"])
    g, f, _ = field(d2q9, g9["prop"], 8, 8)
    tl.bc(f, p, d2q9)
    assert np.array_equal(f.numpy(), g9["bc"])
    out = tl.collide(g9["prop"][:, 3:11, 3:11], p, d2q9)
    assert np.array_equal(out, g9["collide"])
    g, prv, nxt = field(d2q9, g9["prv"], 8, 8)
    tl.propagate_collide_fused(prv, nxt, p, d2q9, (slice(4, 10), slice(5, 9)))
    assert np.array_equal(nxt.numpy(), g9["fused"])


@pytest.mark.parametrize("Np,schedule", [(1, "staged"), (1, "overlapped"), (2, "overlapped"),
                                         (4, "staged")])
def test_d2q9_run_bitwise(d2q9, g9, Np, schedule):
    p = P(g9["params"])
    res = tl.run(tl.SimConfig(Lx=16, Ly=12, model="D2Q9", Np=Np, schedule=schedule, steps=10,
                              params=p, init="random", init_kwargs={"seed": 4}))
    assert np.array_equal(res.populations, g9["run_f10"])


def test_d2q9_reference_properties(d2q9):
    # test_kernels.py:23-33 rest temperature, zero state rejected
    _, _, _, T = tl.moments(d2q9.w[:, None], d2q9)
    assert T[0] == pytest.approx(1 / 3, abs=1e-15)
    with pytest.raises(tl.DegenerateStateError):
        tl.moments(np.zeros((9, 1)), d2q9)
    # test_kernels.py:140-144 momentum exact at order 2
    f = tl.equilibrium(np.float64(1.0), 0.05, 0.0, np.float64(d2q9.cs2), d2q9)
    _, ux, uy, _ = tl.moments(f[:, None], d2q9)
    assert abs(ux[0] - 0.05) < 1e-12 and abs(uy[0]) < 1e-12
    with pytest.raises(tl.DomainError):
        tl.equilibrium(np.float64(-1.0), 0.0, 0.0, np.float64(0.3), d2q9)
    # test_kernels.py:264-269 infinite-tau limit
    rng = np.random.default_rng(13)
    f = 0.2 + rng.random((9, 4))
    out = tl.collide(f, tl.PhysicsParams(tau=1e12), d2q9)
    assert np.allclose(out, f, rtol=1e-11)
    # test_kernels.py:192-197 uniform state invariant under propagate
    g, prv, nxt = field(d2q9, None, 8, 8)
    prv.pops[...] = torch.tensor(d2q9.w)[:, None, None]
    tl.propagate(prv, nxt, d2q9)
    assert torch.equal(nxt.pops[:, 3:11, 3:11], prv.pops[:, 3:11, 3:11])


def test_d2q9_face_plans_and_ring_sentinel(d2q9):
    """test_runtime.py:58-61 and 137-158."""
    plans = tl.face_plans(d2q9)
    assert [len(x) for x in plans[(0, 1)]] == [3, 0, 0]
    assert tl.boundary_bytes_per_site(d2q9) == 24
    tiles = tl.decompose(16, 8, 4, "1d")
    fab = tl.Fabric(4, timeout=5.0)
    ws = [tl.RankWorker(t, d2q9, tl.PhysicsParams(tau=0.8), fab) for t in tiles]
    l = d2q9.find(1, 0)
    g = ws[0].geom
    ws[0].prv.pops[l, g.Hx + g.Lx - 1, g.Hy + 2] = 42.0
    hs = [w._start("x", 0, w.prv) for w in ws]
    for w, h in zip(ws, hs):
        w._finish("x", w.prv, h)
    torch.cuda.synchronize()
    assert ws[1].prv.pops[l, g.Hx - 1, g.Hy + 2].item() == 42.0
    assert ws[2].prv.pops.sum().item() == 0.0


def test_generic_path_equals_specialised_d2q37():
    """The generic per-population kernels reproduce the specialised D2Q37
    kernels bit for bit (both are the reference arithmetic)."""
    vs = tl.build_velocity_set("D2Q37")
    p = tl.PhysicsParams(tau=0.8, gx=1e-5, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                         Twall_bot=1.1 * vs.cs2)
    cfg = dict(Lx=64, Ly=40, steps=6, params=p, init="rayleigh-taylor")
    spec = tl.run(tl.SimConfig(**cfg))
    dev = torch.cuda.current_device()
    _lib.check(_lib.load().tlb_force_generic(dev, 1), "force generic")
    try:
        gen = tl.run(tl.SimConfig(**cfg))
        gen_staged = tl.run(tl.SimConfig(schedule="staged", Np=2, **cfg))
    finally:
        _lib.check(_lib.load().tlb_force_generic(dev, 0), "force generic")
    assert np.array_equal(gen.populations, spec.populations)
    assert np.array_equal(gen_staged.populations, spec.populations)
