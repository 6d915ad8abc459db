"""Parity at the BASELINE.json lattice sizes through size-independent
properties (the CPU oracle needs minutes per step there):

* translation equivariance on the periodic lattice -- shifting the initial
  state by (kx, ky) sites shifts the state after n steps by the same
  amount, bit for bit (every site runs the same IEEE operation sequence);
* rank-count invariance -- 1 tile vs 2 and 4 in-process tiles, bitwise;
* conservation -- total mass and momentum after n periodic, force-free
  steps within 1e-12 relative (reference test_acceptance.py:58-74 bound);
* fast vs exact arithmetic within the north star's 1e-12 relative bound.

C5 = 4096x8192 (configs[4]); C4 = 8192x16384 (configs[3], 80 GB for the
double buffer of one tile) is checked for conservation and fast/exact
agreement on one B200.
"""

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402


@pytest.fixture(scope="module")
def vs():
    return tl.build_velocity_set("D2Q37")


def periodic_worker(vs, Lx, Ly, arith="exact", Np=1, rank=0, fabric=None, gy=0.0):
    p = tl.PhysicsParams(tau=0.8, gy=gy, arith=arith)
    tile = tl.decompose(Lx, Ly, Np, "1d", periodic_y=True)[rank]
    return tl.RankWorker(tile, vs, p, fabric or tl.Fabric(Np), schedule="overlapped",
                         walls=False, periodic_y=True)


def initial_state(vs, Lx, Ly, seed=7):
    macro = tl.init.initial_macro("random", Lx, Ly, vs, seed=seed, amplitude=0.01)
    return tl.equilibrium(*[torch.as_tensor(m).cuda() for m in macro], vs)


def advance(w, f, n):
    w.load_block(f)
    w.run_steps(0, n)
    out = w.physical_block()
    w.collect()
    return out


def macro_contract(vs, fast, exact):
    """SURVEY §8c between two (Q, ...) device blocks: f, rho and T within
    1e-12 relative, |du| <= 1e-12 * cs (moments on the device, exact
    arithmetic)."""
    rel_f = ((fast - exact).abs() / exact.abs()).max().item()
    mf, me = tl.moments(fast, vs), tl.moments(exact, vs)
    rel_rho = ((mf[0] - me[0]).abs() / me[0]).max().item()
    rel_T = ((mf[3] - me[3]).abs() / me[3]).max().item()
    du = torch.hypot(mf[1] - me[1], mf[2] - me[2]).max().item() / vs.cs2 ** 0.5
    assert rel_f <= 1e-12 and rel_rho <= 1e-12 and rel_T <= 1e-12 and du <= 1e-12, \
        (rel_f, rel_rho, rel_T, du)
    return rel_f, rel_rho, rel_T, du


def test_c5_translation_equivariance_and_fast_vs_exact(vs):
    Lx, Ly, n = 4096, 8192, 4
    f0 = initial_state(vs, Lx, Ly)
    w = periodic_worker(vs, Lx, Ly)
    ref = advance(w, f0, n)
    for kx, ky in [(1, 0), (3, 5), (-1234, 777)]:
        shifted = advance(w, torch.roll(f0, shifts=(kx, ky), dims=(1, 2)), n)
        assert torch.equal(shifted, torch.roll(ref, shifts=(kx, ky), dims=(1, 2))), (kx, ky)
        del shifted
    del w
    wf = periodic_worker(vs, Lx, Ly, arith="fast")
    fast = advance(wf, f0, n)
    print("C5 fast vs exact (f, rho, T, |du|/cs):", macro_contract(vs, fast, ref))


def test_c5_rank_count_invariance(vs):
    Lx, Ly, n = 4096, 8192, 3
    f0 = initial_state(vs, Lx, Ly, seed=11)
    one = advance(periodic_worker(vs, Lx, Ly), f0, n)
    for Np in (2, 4):
        fab = tl.Fabric(Np)
        ws = [periodic_worker(vs, Lx, Ly, Np=Np, rank=r, fabric=fab) for r in range(Np)]
        for w in ws:
            t = w.tile
            w.load_block(f0[:, t.x0:t.x0 + t.Lx, t.y0:t.y0 + t.Ly].contiguous())
        for s in range(n):
            for phase in ("step_begin", "step_mid", "step_end"):
                for w in ws:
                    getattr(w, phase)(s)
        for w in ws:
            t = w.tile
            assert torch.equal(w.physical_block(), one[:, t.x0:t.x0 + t.Lx, t.y0:t.y0 + t.Ly])
            w.collect()
        del ws


def _totals(vs, f):
    c = torch.tensor(vs.c, dtype=torch.float64, device=f.device)
    per_q = f.sum(dim=(1, 2))
    return per_q.sum().item(), (c[:, 0] @ per_q).item(), (c[:, 1] @ per_q).item()


def test_c4_conservation_and_fast_vs_exact(vs):
    """C4 on one GPU: 80 GB double buffer + one 40 GB initial state; the
    fast/exact comparison uses every 97th column (0.4 GB) so that two full
    40 GB result copies are never resident together."""
    Lx, Ly, n = 8192, 16384, 3
    import gc
    gc.collect()
    torch.cuda.empty_cache()          # blocks cached by the C5 tests
    free, _ = torch.cuda.mem_get_info()
    if free < 130e9:
        pytest.skip(f"needs ~130 GB of free HBM (C4 on one GPU), {free / 1e9:.0f} GB free")
    w = periodic_worker(vs, Lx, Ly)
    g = w.geom

    def run_from_seed(arith):
        w.tparams = tl._lib.params(tl.PhysicsParams(tau=0.8, arith=arith), vs)
        w._graphs.clear()
        f0 = initial_state(vs, Lx, Ly, seed=3)
        before = _totals(vs, f0)
        w.load_block(f0)
        del f0
        torch.cuda.empty_cache()
        w.run_steps(0, n)
        w.collect()
        return before, w.prv.pops[:, g.phys_x, g.phys_y]

    (m0, px0, py0), view = run_from_seed("exact")
    m1, px1, py1 = _totals(vs, view)
    assert abs(m1 - m0) / m0 < 1e-12
    assert abs(px1 - px0) / m0 < 1e-12 and abs(py1 - py0) / m0 < 1e-12
    sample = view[:, ::97, :].clone()
    _, view = run_from_seed("fast")
    print("C4 fast vs exact (f, rho, T, |du|/cs):",
          macro_contract(vs, view[:, ::97, :].clone(), sample))
