"""The reference's acceptance and property tests, run on the CUDA path.

Mirrors /root/reference/pkg/tests/test_acceptance.py (c02-c05, c10, c11),
test_kernels.py (collide/propagate/bc properties) and test_runtime.py (step,
snapshots, metrics) -- same inputs, same tolerances -- plus layout and API
checks of the drop-in.
"""

import numpy as np
import pytest

from conftest import periodic_fill, random_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402


@pytest.fixture(scope="module")
def vs():
    return tl.build_velocity_set("D2Q37")


def dev_field(vs, Lx, Ly, state=None, layout=tl.SOA):
    g = tl.LatticeGeometry(Lx, Ly, 3, 3, 37, layout)
    prv, nxt = tl.allocate_field(g, vs)
    if state is not None:
        prv.pops.copy_(torch.as_tensor(state))
    return g, prv, nxt


# ------------------------------------------------------ acceptance c02-c05 --

def test_c02_conservation_500_steps(vs):
    """test_acceptance.py:58-74: mass/momentum drift < 1e-12 over 500 steps."""
    cfg = tl.SimConfig(Lx=64, Ly=64, Np=1, tiling="1d", schedule="overlapped",
                       steps=500, params=tl.PhysicsParams(tau=0.8), walls=False,
                       periodic_y=True, init="random", init_kwargs={"seed": 7})
    rho, ux, uy, T = tl.init.random_near_equilibrium_macro(64, 64, vs, seed=7)
    f0 = tl.equilibrium(rho, ux, uy, T, vs)
    res = tl.run(cfg)
    c = vs.c.astype(float)
    mass0, mass1 = f0.sum(), res.populations.sum()
    assert abs(mass1 - mass0) / mass0 < 1e-12
    for axis in (0, 1):
        p0 = float(np.einsum("l,lxy->", c[:, axis], f0))
        p1 = float(np.einsum("l,lxy->", c[:, axis], res.populations))
        assert abs(p1 - p0) / mass0 < 1e-12


def test_c03_propagate_permutation(vs):
    """test_acceptance.py:77-87."""
    g, prv, nxt = dev_field(vs, 32, 32)
    st = random_state(g.NX, g.NY, seed=11)
    prv.pops.copy_(torch.as_tensor(st))
    periodic_fill(prv.pops)
    tl.propagate(prv, nxt, vs)
    before = np.sort(prv.numpy()[:, 3:35, 3:35].reshape(-1))
    after = np.sort(nxt.numpy()[:, 3:35, 3:35].reshape(-1))
    assert np.array_equal(before, after)


def test_c04_fused_equivalence_100_states(vs):
    """test_acceptance.py:90-103: fused == propagate -> collide, bitwise."""
    params = tl.PhysicsParams(tau=0.8, gy=-1e-4)
    g = tl.LatticeGeometry(16, 16, 3, 3, 37)
    prv, nxt = tl.allocate_field(g, vs)
    ref = tl.PopulationField(g, "nxt")
    region = (g.phys_x, g.phys_y)
    for seed in range(100):
        prv.pops.copy_(torch.as_tensor(random_state(g.NX, g.NY, seed=seed)))
        tl.propagate(prv, ref, vs, region)
        blk = tl.collide(ref.pops[:, g.phys_x, g.phys_y], params, vs)
        tl.propagate_collide_fused(prv, nxt, params, vs, region)
        assert torch.equal(nxt.pops[:, g.phys_x, g.phys_y], blk), seed


def test_c05_rank_count_invariance(vs):
    """test_acceptance.py:106-121 (1-D variants; 2-D tilings are out of scope)."""
    p = tl.PhysicsParams(tau=0.8, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    kw = dict(Lx=128, Ly=128, model="D2Q37", steps=100, params=p, init="random",
              init_kwargs={"seed": 3})
    ref = tl.run(tl.SimConfig(Np=1, schedule="staged", **kw))
    for Np, schedule in ((4, "overlapped"), (4, "staged"), (8, "overlapped"), (2, "staged")):
        res = tl.run(tl.SimConfig(Np=Np, tiling="1d", schedule=schedule, **kw))
        assert np.array_equal(res.populations, ref.populations), (Np, schedule)


def test_c10_bc_contract(vs):
    """test_acceptance.py:200-216."""
    g, f, _ = dev_field(vs, 12, 16, random_state(18, 22, seed=5))
    params = tl.PhysicsParams(tau=0.9, Twall_top=0.62, Twall_bot=0.81)
    interior = f.numpy()[:, g.phys_x, g.Hy + 3:g.Hy + g.Ly - 3].copy()
    tl.bc(f, params, vs)
    for rows, Twall in ((slice(g.Hy + g.Ly - 3, g.Hy + g.Ly), 0.62),
                        (slice(g.Hy, g.Hy + 3), 0.81)):
        _, ux, uy, T = tl.moments(f.pops[:, g.phys_x, rows], vs)
        assert max(ux.abs().max().item(), uy.abs().max().item()) < 1e-14
        assert (T - Twall).abs().max().item() < 1e-12
    assert np.array_equal(f.numpy()[:, g.phys_x, g.Hy + 3:g.Hy + g.Ly - 3], interior)


@pytest.mark.parametrize("schedule", ["overlapped", "staged"])
def test_c11_halo_poisoning(vs, schedule):
    """test_acceptance.py:219-230 (1-D tiling): NaN halos never reach physics."""
    p = tl.PhysicsParams(tau=0.8, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    res = tl.run(tl.SimConfig(Lx=32, Ly=32, Np=4, tiling="1d", schedule=schedule,
                              steps=50, params=p, init="random",
                              init_kwargs={"seed": 2}, debug_poison=True))
    assert np.all(np.isfinite(res.populations))


# ---------------------------------------------------- kernel properties --

def test_collide_fixed_point(vs):
    """test_kernels.py:242-249."""
    rho = np.full((3,), 1.1)
    feq = tl.equilibrium(rho, np.full((3,), 0.02), np.zeros(3), np.full((3,), vs.cs2), vs)
    for arith in ("exact", "fast"):
        out = tl.collide(feq, tl.PhysicsParams(tau=0.9, arith=arith), vs)
        assert np.allclose(out, feq, rtol=1e-12, atol=1e-15)


def test_collide_conserves_mass_momentum(vs):
    """test_kernels.py:252-262."""
    rng = np.random.default_rng(11)
    f = 0.2 + rng.random((37, 5))
    c = vs.c.astype(float)
    for arith in ("exact", "fast"):
        out = tl.collide(f, tl.PhysicsParams(tau=0.7, arith=arith), vs)
        for j in range(5):
            assert out[:, j].sum() == pytest.approx(f[:, j].sum(), rel=1e-12)
            for axis in (0, 1):
                assert (c[:, axis] * out[:, j]).sum() == pytest.approx(
                    (c[:, axis] * f[:, j]).sum(), rel=1e-10, abs=1e-12)


def test_collide_is_contraction(vs):
    """test_kernels.py:273-282: ||f' - feq|| = |1 - 1/tau| ||f - feq||."""
    rng = np.random.default_rng(17)
    f = 0.2 + rng.random((37, 6))
    rho, ux, uy, T = tl.moments(f, vs)
    feq = tl.equilibrium(rho, ux, uy, T, vs)
    out = tl.collide(f, tl.PhysicsParams(tau=0.8), vs)
    lhs = np.linalg.norm(out - feq)
    rhs = abs(1 - 1 / 0.8) * np.linalg.norm(f - feq)
    assert lhs == pytest.approx(rhs, rel=1e-12)


def test_propagate_moves_single_value(vs):
    """test_kernels.py:183-189."""
    g, prv, nxt = dev_field(vs, 8, 8)
    l = vs.find(2, 1)
    prv.pops[l, g.Hx + 4, g.Hy + 4] = 1.0
    tl.propagate(prv, nxt, vs)
    assert nxt.pops[l, g.Hx + 6, g.Hy + 5].item() == 1.0
    assert nxt.pops[l].sum().item() == 1.0


def test_equilibrium_mass_and_tensor_oracle(vs):
    """test_kernels.py:110-121 / 129-137 (independent tensor oracle)."""
    import itertools
    rng = np.random.default_rng(5)
    cs = np.sqrt(vs.cs2)
    d = np.eye(2)
    for _ in range(10):
        rho = 0.5 + rng.random()
        u = 0.1 * rng.standard_normal(2)
        T = vs.cs2 * (0.8 + 0.4 * rng.random())
        got = tl.equilibrium(np.float64(rho), u[0], u[1], np.float64(T), vs)
        v = u / cs
        th = T / vs.cs2 - 1.0
        want = np.empty(37)
        for l in range(37):
            e = vs.c[l] / cs
            term = 1.0 + e @ v + 0.5 * np.tensordot(np.outer(v, v) + th * d, np.outer(e, e) - d)
            a3 = np.zeros((2, 2, 2)); h3 = np.zeros((2, 2, 2))
            a4 = np.zeros((2, 2, 2, 2)); h4 = np.zeros((2, 2, 2, 2))
            for i, j, k in itertools.product(range(2), repeat=3):
                a3[i, j, k] = v[i]*v[j]*v[k] + th*(d[i, j]*v[k] + d[i, k]*v[j] + d[j, k]*v[i])
                h3[i, j, k] = e[i]*e[j]*e[k] - (d[i, j]*e[k] + d[i, k]*e[j] + d[j, k]*e[i])
            for i, j, k, m in itertools.product(range(2), repeat=4):
                a4[i, j, k, m] = (v[i]*v[j]*v[k]*v[m]
                                  + th*(d[i, j]*v[k]*v[m] + d[i, k]*v[j]*v[m] + d[i, m]*v[j]*v[k]
                                        + d[j, k]*v[i]*v[m] + d[j, m]*v[i]*v[k] + d[k, m]*v[i]*v[j])
                                  + th**2*(d[i, j]*d[k, m] + d[i, k]*d[j, m] + d[i, m]*d[j, k]))
                h4[i, j, k, m] = (e[i]*e[j]*e[k]*e[m]
                                  - (d[i, j]*e[k]*e[m] + d[i, k]*e[j]*e[m] + d[i, m]*e[j]*e[k]
                                     + d[j, k]*e[i]*e[m] + d[j, m]*e[i]*e[k] + d[k, m]*e[i]*e[j])
                                  + (d[i, j]*d[k, m] + d[i, k]*d[j, m] + d[i, m]*d[j, k]))
            term += np.sum(a3 * h3) / 6.0 + np.sum(a4 * h4) / 24.0
            want[l] = vs.w[l] * rho * term
        assert np.allclose(got, want, rtol=1e-13, atol=1e-16)
        assert got.sum() == pytest.approx(rho, rel=1e-13)


# ---------------------------------------------------------- run / runtime --

def test_uniform_equilibrium_fixed_point(vs):
    """test_runtime.py:219-230."""
    cs2 = vs.cs2
    res = tl.run(tl.SimConfig(Lx=16, Ly=16, Np=2, tiling="1d", schedule="staged", steps=5,
                              params=tl.PhysicsParams(tau=0.8, Twall_top=cs2, Twall_bot=cs2),
                              init="uniform"))
    assert np.max(np.abs(res.macro.rho - 1.0)) < 1e-12
    assert np.max(np.abs(res.macro.T - cs2)) < 1e-12
    assert np.max(np.abs(res.macro.ux)) < 1e-13
    assert np.max(np.abs(res.macro.uy)) < 1e-13


def test_zero_steps_returns_initial_state(vs):
    """test_runtime.py:233-239."""
    res = tl.run(tl.SimConfig(Lx=8, Ly=8, Np=1, steps=0, init="uniform"))
    want = np.broadcast_to(vs.w[:, None, None], (37, 8, 8))
    assert np.allclose(res.populations, want, rtol=1e-14)
    assert res.mlups == 0.0


def test_metrics_and_snapshots(vs):
    """test_runtime.py:271-288."""
    res = tl.run(tl.SimConfig(Lx=16, Ly=8, Np=2, tiling="1d", steps=4, snapshot_every=2,
                              params=tl.PhysicsParams(tau=0.9)))
    assert len(res.metrics) == 4 * 2
    for key in ("step", "rank", "t_comm_nc", "t_comm_c", "t_bulk", "t_border", "negatives"):
        assert key in res.metrics[0]
    assert res.mlups > 0.0 and res.wall_seconds > 0.0
    assert [s for s, _ in res.snapshots] == [2, 4]
    assert res.snapshots[0][1].rho.shape == (16, 8)


def test_staged_equals_overlapped(vs):
    """test_runtime.py:242-249 (1-D)."""
    p = tl.PhysicsParams(tau=0.8, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    kw = dict(Lx=16, Ly=16, Np=4, tiling="1d", steps=8, params=p, init="random",
              init_kwargs={"seed": 3})
    a = tl.run(tl.SimConfig(schedule="staged", **kw))
    b = tl.run(tl.SimConfig(schedule="overlapped", **kw))
    assert np.array_equal(a.populations, b.populations)


@pytest.mark.parametrize("tiling,periodic", [("1d", False), ((2, 2), False), ("1d", True)])
def test_layouts_same_bits(vs, tiling, periodic):
    """Layouts are storage only: AoS and column fields give the SoA bits
    (geometry.py:1-7), through the halo exchange of 2 or 4 ranks."""
    p = tl.PhysicsParams(tau=0.8, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    kw = dict(Lx=24, Ly=20, Np=2 if tiling == "1d" else 4, tiling=tiling, steps=5, params=p,
              init="random", init_kwargs={"seed": 9}, walls=not periodic, periodic_y=periodic)
    a = tl.run(tl.SimConfig(layout="soa", **kw))
    for layout in ("aos", "column"):
        b = tl.run(tl.SimConfig(layout=layout, **kw))
        assert np.array_equal(a.populations, b.populations), layout


def test_field_layout_conversion_round_trip(vs):
    g = tl.LatticeGeometry(6, 5, 3, 3, 37)
    f, _ = tl.allocate_field(g, vs)
    f.pops.copy_(torch.randn(f.pops.shape, dtype=torch.float64, device=f.device))
    for layout in (tl.AOS, tl.COLUMN):
        c = f.converted(layout)
        assert c.geom.layout == layout and torch.equal(c.pops, f.pops)
        flat = c.flat
        for (l, x, y) in [(0, 0, 0), (5, 2, 7), (36, 11, 10)]:
            assert flat[tl.site_index(c.geom, l, x, y)].item() == f.pops[l, x, y].item()
        assert torch.equal(c.converted(tl.SOA).data, f.data)


def test_device_output_and_explicit_f0(vs):
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    host = tl.run(tl.SimConfig(Lx=32, Ly=16, steps=3, params=p, init="rayleigh-taylor"))
    f0 = tl.init.build_initial_state("rayleigh-taylor", 32, 16, vs)
    dev = tl.run(tl.SimConfig(Lx=32, Ly=16, steps=3, params=p, output="device"), f0=f0)
    assert dev.populations.is_cuda
    assert np.array_equal(dev.populations.cpu().numpy(), host.populations)


# ------------------------------------------------------------ 2-D tiling --

@pytest.mark.parametrize("tiling,schedule", [((2, 2), "overlapped"), ((2, 2), "staged"),
                                             ((2, 4), "overlapped"), ((1, 4), "staged"),
                                             ((4, 2), "overlapped")])
def test_2d_rank_invariance(vs, tiling, schedule):
    """test_acceptance.py:106-121 / test_runtime.py:252-260 with 2-D grids:
    bitwise equal to one rank (walls in Y, periodic X)."""
    p = tl.PhysicsParams(tau=0.8, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    kw = dict(Lx=64, Ly=48, model="D2Q37", steps=12, params=p, init="random",
              init_kwargs={"seed": 5})
    ref = tl.run(tl.SimConfig(Np=1, schedule="staged", **kw))
    Np = tiling[0] * tiling[1]
    res = tl.run(tl.SimConfig(Np=Np, tiling=tiling, schedule=schedule, **kw))
    assert np.array_equal(res.populations, ref.populations)


@pytest.mark.parametrize("schedule", ["overlapped", "staged"])
def test_2d_periodic_y_invariance(vs, schedule):
    p = tl.PhysicsParams(tau=0.8, gx=1e-5)
    kw = dict(Lx=32, Ly=32, steps=10, params=p, walls=False, periodic_y=True,
              init="random", init_kwargs={"seed": 8})
    ref = tl.run(tl.SimConfig(Np=1, schedule="staged", **kw))
    for tiling in ((2, 2), (1, 2), (2, 4)):
        Np = tiling[0] * tiling[1]
        res = tl.run(tl.SimConfig(Np=Np, tiling=tiling, schedule=schedule, **kw))
        assert np.array_equal(res.populations, ref.populations), tiling


def test_2d_halo_poisoning(vs):
    """test_acceptance.py:219-230 with the reference's 2x2 grid."""
    p = tl.PhysicsParams(tau=0.8, gy=-1e-4, Twall_top=0.6, Twall_bot=0.75)
    for schedule in ("overlapped", "staged"):
        res = tl.run(tl.SimConfig(Lx=32, Ly=32, Np=4, tiling=(2, 2), schedule=schedule,
                                  steps=20, params=p, init="random",
                                  init_kwargs={"seed": 2}, debug_poison=True))
        assert np.all(np.isfinite(res.populations))


def _workers(vs, Lx, Ly, Np, tiling, periodic_y=False, walls=True):
    tiles = tl.decompose(Lx, Ly, Np, tiling, periodic_y=periodic_y)
    fab = tl.Fabric(Np, timeout=5.0)
    p = tl.PhysicsParams(tau=0.8, Twall_top=0.6, Twall_bot=0.8)
    return [tl.RankWorker(t, vs, p, fab, walls=walls, periodic_y=periodic_y) for t in tiles]


def test_corner_diagonal_via_protocol_order(vs):
    """test_runtime.py:161-185: Y exchange first, then X over the full
    height, so a corner sentinel from the diagonal neighbour arrives."""
    ws = _workers(vs, 8, 8, 4, (2, 2), periodic_y=True, walls=False)
    l = vs.find(-1, -1)
    g = ws[0].geom
    ws[3].prv.pops[l, g.Hx, g.Hy] = 7.0       # rank 3 is up-right of rank 0
    hs = [w._start("y", 0, w.prv) for w in ws]
    for w, h in zip(ws, hs):
        w._finish("y", w.prv, h)
    hs = [w._start("x", 0, w.prv) for w in ws]
    for w, h in zip(ws, hs):
        w._finish("x", w.prv, h)
    torch.cuda.synchronize()
    assert ws[0].prv.pops[l, g.Hx + g.Lx, g.Hy + g.Ly].item() == 7.0


def test_wall_rank_outer_halo_untouched_by_exchange(vs):
    """test_runtime.py:188-214."""
    ws = _workers(vs, 8, 8, 2, (1, 2))
    for w in ws:
        g = w.geom
        blk = torch.arange(37 * g.Lx * g.Ly, dtype=torch.float64, device="cuda").reshape(
            37, g.Lx, g.Ly) + 1000.0 * (w.tile.rank + 1)
        w.prv.pops.zero_()
        w.prv.pops[:, g.phys_x, g.phys_y] = blk
        w._extend_wall_halos(w.prv)
    torch.cuda.synchronize()
    g = ws[0].geom
    lo = ws[0].prv.pops[:, g.phys_x, g.Hy].clone()
    hi = ws[1].prv.pops[:, g.phys_x, g.Hy + g.Ly - 1].clone()
    hs = [w._start("y", 0, w.prv) for w in ws]
    for w, h in zip(ws, hs):
        w._finish("y", w.prv, h)
    hs = [w._start("x", 0, w.prv) for w in ws]
    for w, h in zip(ws, hs):
        w._finish("x", w.prv, h)
    torch.cuda.synchronize()
    for k in range(g.Hy):
        assert torch.equal(ws[0].prv.pops[:, g.phys_x, k], lo)
        assert torch.equal(ws[1].prv.pops[:, g.phys_x, g.Hy + g.Ly + k], hi)


def test_pgm_bytes_match_reference(tmp_path):
    """io.write_pgm (io.py:13-24) on the device: byte-identical image."""
    from conftest import golden
    from paper_1703_00185_b200 import io as tio
    g = golden("io.npz")
    tio.write_pgm(tmp_path / "t.pgm", g["T"])
    assert (tmp_path / "t.pgm").read_bytes() == g["pgm"].tobytes()
    # a device (strided) view gives the same bytes
    t = torch.as_tensor(np.pad(g["T"], ((0, 0), (3, 3)))).cuda()[:, 3:-3]
    assert tio.pgm_bytes(t) == g["pgm"].tobytes()


# ------------------------------------------------------ CUDA-graph replay --

def _single_worker(vs, schedule, walls, arith="exact"):
    p = tl.PhysicsParams(tau=0.8, gx=1e-6, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                         Twall_bot=1.1 * vs.cs2, arith=arith)
    tile = tl.decompose(48, 40, 1, "1d", periodic_y=not walls)[0]
    w = tl.RankWorker(tile, vs, p, tl.Fabric(1), schedule=schedule, walls=walls,
                      periodic_y=not walls)
    macro = tl.init.initial_macro("random", 48, 40, vs, seed=5)
    w.load_block(tl.equilibrium(*[torch.as_tensor(m).cuda() for m in macro], vs))
    return w


@pytest.mark.parametrize("schedule,walls", [("overlapped", True), ("staged", True),
                                            ("overlapped", False), ("staged", False)])
def test_graph_replay_equals_step_loop(vs, schedule, walls):
    """RankWorker.run_steps (CUDA graphs of 32 steps) gives the bits and the
    per-step negatives of the plain step() loop, across graph boundaries and
    for both buffer parities."""
    a, b = _single_worker(vs, schedule, walls), _single_worker(vs, schedule, walls)
    assert b.graphable()
    for s in range(3 + 70 + 40):
        a.step(s)
    b.run_steps(0, 3)          # odd prefix: the graphs start on the other parity
    b.run_steps(3, 69)         # 64 replayed + 5 plain -> even again
    b.run_steps(72, 41)        # 32 replayed on the first parity + 9 plain
    assert torch.equal(a.physical_block(), b.physical_block())
    ma, mb = a.metrics, b.metrics
    assert [m["negatives"] for m in ma] == [m["negatives"] for m in mb]
    assert len(b._graphs) == 2
    # replayed steps report the block's average step time
    replayed = [m["t_bulk"] for m in mb[3:3 + 64]]
    assert all(np.isfinite(t) and t > 0 for t in replayed)


def test_graph_replay_reports_failures_with_step(vs):
    """A degenerate state is reported from inside a replayed graph with the
    same step number as the step() loop (collect -> DegenerateStateError)."""
    errs = []
    for graphed in (False, True):
        w = _single_worker(vs, "overlapped", True)
        f = w.physical_block()
        f[:, 20:24, 10:14] *= -1.0          # negative density in a patch
        w.load_block(f)
        if graphed:
            w.run_steps(0, 64)
        else:
            for s in range(64):
                w.step(s)
        with pytest.raises(tl.DegenerateStateError) as e:
            w.collect()
        errs.append(str(e.value).split(":")[0])
        x, y = e.value.sites[0]          # padded coordinates, first site flagged
        assert 23 <= x < 27 and 13 <= y < 17
    assert errs[0] == errs[1] == "rank 0 step 0"


def test_run_uses_graphs_and_matches_multi_rank(vs):
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    kw = dict(Lx=64, Ly=32, steps=100, params=p, init="rayleigh-taylor", snapshot_every=40)
    one = tl.run(tl.SimConfig(Np=1, **kw))
    two = tl.run(tl.SimConfig(Np=2, **kw))
    assert np.array_equal(one.populations, two.populations)
    assert [s for s, _ in one.snapshots] == [40, 80] == [s for s, _ in two.snapshots]
    for (_, a), (_, b) in zip(one.snapshots, two.snapshots):
        for name in ("rho", "ux", "uy", "T"):
            assert np.array_equal(np.asarray(getattr(a, name)), np.asarray(getattr(b, name)))
    assert len(one.metrics) == 100
