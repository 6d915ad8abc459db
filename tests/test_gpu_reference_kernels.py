"""The reference's kernel unit tests (tests/test_kernels.py), one for one,
run against the CUDA kernels through the drop-in API.

Each test keeps the reference test's name, inputs and tolerance and cites
its lines; the four that already live in test_gpu_acceptance.py under the
same name (propagate_moves_single_value, collide_fixed_point,
collide_conserves_mass_momentum, collide_is_contraction) are not repeated.
Fields are CUDA tensors here, so element access goes through torch.
"""

import itertools

import numpy as np
import pytest

from conftest import periodic_fill, random_state

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402


@pytest.fixture(scope="module")
def d2q37():
    return tl.build_velocity_set("D2Q37")


@pytest.fixture(scope="module")
def d2q9():
    return tl.build_velocity_set("D2Q9")


def pair(vs, Lx=8, Ly=8):
    g = tl.LatticeGeometry(Lx, Ly, 3, 3, vs.Q)
    prv, nxt = tl.allocate_field(g, vs)
    return g, prv, nxt


def fill_random(field, vs, seed):
    g = field.geom
    field.pops.copy_(torch.as_tensor(random_state(g.NX, g.NY, seed=seed, Q=vs.Q)))


# ----------------------------------------------------------------- moments --

def test_moments_rest_state(d2q37):
    """test_kernels.py:16-20."""
    rho, ux, uy, T = tl.moments(d2q37.w[:, None], d2q37)
    assert rho[0] == pytest.approx(1.0, abs=1e-14)
    assert abs(ux[0]) < 1e-14 and abs(uy[0]) < 1e-14
    assert T[0] == pytest.approx(d2q37.cs2, abs=1e-13)


def test_moments_d2q9_rest_temperature(d2q9):
    """test_kernels.py:23-28: T at rest = sum_l w_l |c_l|^2 / 2 = 1/3."""
    c2 = (d2q9.c.astype(float) ** 2).sum(axis=1)
    expect = float(np.dot(d2q9.w, c2)) / 2.0
    T = tl.moments(d2q9.w[:, None], d2q9)[3]
    assert expect == pytest.approx(1 / 3, abs=1e-15)
    assert T[0] == pytest.approx(expect, abs=1e-15)


def test_moments_zero_state_rejected(d2q9):
    """test_kernels.py:31-33."""
    with pytest.raises(tl.DegenerateStateError):
        tl.moments(np.zeros((9, 1)), d2q9)


def test_moments_match_brute_force(d2q37):
    """test_kernels.py:36-48: per-site sums against a direct evaluation."""
    f = 0.1 + np.random.default_rng(2).random((37, 4))
    rho, ux, uy, T = tl.moments(f, d2q37)
    c = d2q37.c.astype(float)
    for j in range(4):
        col = f[:, j]
        r = col.sum()
        u = c.T @ col / r
        peculiar = ((c - u) ** 2).sum(axis=1)
        assert rho[j] == pytest.approx(r, rel=1e-14)
        assert ux[j] == pytest.approx(u[0], rel=1e-12)
        assert T[j] == pytest.approx(float(peculiar @ col) / (2 * r), rel=1e-11)


# ------------------------------------------------------------- equilibrium --

def _sym(*parts):
    """Sum of the distinct index placements of outer products of `parts`
    over 3 or 4 indices (the delta-symmetrised Hermite terms)."""
    n = sum(p.ndim for p in parts)
    letters = "ijkm"[:n]
    seen, total = set(), 0
    for perm in itertools.permutations(range(n)):
        idx, k = [], 0
        for p in parts:
            idx.append("".join(letters[perm[k + t]] for t in range(p.ndim)))
            k += p.ndim
        key = tuple(frozenset(s) for s in idx)
        if all(p is parts[0] for p in parts):   # identical factors commute
            key = frozenset(key)
        if key in seen:
            continue
        seen.add(key)
        total = total + np.einsum(",".join(idx) + "->" + letters, *parts)
    return total


def hermite_tensor(rho, u, T, vs, order):
    """Independent tensor-contraction evaluation of the order-N Hermite
    equilibrium (the reference's hermite_oracle, test_kernels.py:53-108)."""
    cs = np.sqrt(vs.cs2)
    v = np.asarray(u, dtype=float) / cs
    th = T / vs.cs2 - 1.0
    d = np.eye(2)
    out = np.empty(vs.Q)
    for l in range(vs.Q):
        e = vs.c[l] / cs
        val = 1.0 + e @ v
        if order >= 2:
            val += 0.5 * np.sum((np.outer(v, v) + th * d) * (np.outer(e, e) - d))
        if order >= 3:
            a3 = np.einsum("i,j,k->ijk", v, v, v) + th * _sym(d, v)
            h3 = np.einsum("i,j,k->ijk", e, e, e) - _sym(d, e)
            val += np.sum(a3 * h3) / 6.0
        if order >= 4:
            vv, ee = np.outer(v, v), np.outer(e, e)
            a4 = np.einsum("i,j,k,m->ijkm", v, v, v, v) + th * _sym(d, vv) + th ** 2 * _sym(d, d)
            h4 = np.einsum("i,j,k,m->ijkm", e, e, e, e) - _sym(d, ee) + _sym(d, d)
            val += np.sum(a4 * h4) / 24.0
        out[l] = vs.w[l] * rho * val
    return out


def test_sym_counts():
    d, v = np.eye(2), np.array([0.3, -0.7])
    # 3 placements of delta x vector, 6 of delta x (v v), 3 of delta x delta
    assert np.allclose(_sym(d, v)[0, 0, 0], 3 * v[0])
    assert np.allclose(_sym(d, np.outer(v, v))[0, 0, 0, 0], 6 * v[0] ** 2)
    assert np.allclose(_sym(d, d)[0, 0, 0, 0], 3.0)
    assert np.allclose(_sym(d, d)[0, 0, 1, 1], 1.0)


@pytest.mark.parametrize("model,order", [("D2Q37", 4), ("D2Q9", 2)])
def test_equilibrium_matches_tensor_oracle(model, order, d2q37, d2q9):
    """test_kernels.py:110-121 (rtol 1e-13, atol 1e-16)."""
    vs = d2q37 if model == "D2Q37" else d2q9
    rng = np.random.default_rng(5)
    for _ in range(10):
        rho = 0.5 + rng.random()
        u = 0.1 * rng.standard_normal(2)
        T = vs.cs2 * (0.8 + 0.4 * rng.random())
        got = tl.equilibrium(np.float64(rho), u[0], u[1], np.float64(T), vs, order=order)
        assert np.allclose(got, hermite_tensor(rho, u, T, vs, order), rtol=1e-13, atol=1e-16)


def test_equilibrium_mass_preserved(d2q37):
    """test_kernels.py:129-137."""
    rng = np.random.default_rng(9)
    for _ in range(5):
        rho = 0.5 + rng.random()
        f = tl.equilibrium(np.float64(rho), 0.08 * rng.standard_normal(),
                           0.08 * rng.standard_normal(),
                           np.float64(d2q37.cs2 * (0.9 + 0.2 * rng.random())), d2q37)
        assert f.sum() == pytest.approx(rho, rel=1e-13)


def test_equilibrium_momentum_exact_d2q9(d2q9):
    """test_kernels.py:140-144."""
    f = tl.equilibrium(np.float64(1.0), 0.05, 0.0, np.float64(d2q9.cs2), d2q9)
    _, ux, uy, _ = tl.moments(f[:, None], d2q9)
    assert abs(ux[0] - 0.05) < 1e-12 and abs(uy[0]) < 1e-12


def test_equilibrium_rejects_bad_state(d2q9):
    """test_kernels.py:147-151: negative density, zero temperature."""
    for rho, T in ((-1.0, 0.3), (1.0, 0.0)):
        with pytest.raises(tl.DomainError):
            tl.equilibrium(np.float64(rho), 0.0, 0.0, np.float64(T), d2q9)


# ------------------------------------------------------------- apply_shift --

def _shifted(u, v, T, **params):
    return tuple(float(a) for a in tl.apply_shift(u, v, T, tl.PhysicsParams(**params)))


def test_shift_identity_without_force():
    """test_kernels.py:156-159: no force, no shift (bit for bit)."""
    assert _shifted(0.1, -0.2, 0.5, tau=1.0) == (0.1, -0.2, 0.5)


def test_shift_formula():
    """test_kernels.py:162-167: u + tau g, T - tau^2 g^2 / D."""
    got = _shifted(0.0, 0.0, 0.5, tau=1.0, gy=-0.01)
    assert got[0] == 0.0
    assert got[1:] == (pytest.approx(-0.01), pytest.approx(0.5 - 5e-5))


def test_shift_rejects_frozen_temperature():
    """test_kernels.py:170-173."""
    with pytest.raises(tl.DomainError):
        tl.apply_shift(0.0, 0.0, 0.5, tl.PhysicsParams(tau=10.0, gy=-0.5))


# --------------------------------------------------------------- propagate --

def test_propagate_uniform_invariant(d2q9):
    """test_kernels.py:192-197."""
    g, prv, nxt = pair(d2q9)
    prv.pops[...] = torch.tensor(d2q9.w)[:, None, None]
    tl.propagate(prv, nxt, d2q9)
    assert torch.equal(nxt.pops[:, g.phys_x, g.phys_y], prv.pops[:, g.phys_x, g.phys_y])


def test_propagate_is_permutation(d2q37):
    """test_kernels.py:200-209: on a periodic lattice the physical values
    are only permuted."""
    g, prv, nxt = pair(d2q37)
    fill_random(prv, d2q37, seed=0)
    periodic_fill(prv.pops)
    tl.propagate(prv, nxt, d2q37)
    before = torch.sort(prv.pops[:, g.phys_x, g.phys_y].reshape(-1)).values
    after = torch.sort(nxt.pops[:, g.phys_x, g.phys_y].reshape(-1)).values
    assert torch.equal(before, after)


def test_propagate_region_must_be_physical(d2q9):
    """test_kernels.py:212-215."""
    g, prv, nxt = pair(d2q9)
    with pytest.raises(tl.ContractViolation):
        tl.propagate(prv, nxt, d2q9, (slice(0, g.NX), g.phys_y))


# ---------------------------------------------------------------------- bc --

def test_bc_wall_moments(d2q37):
    """test_kernels.py:220-237: wall rows at rest at the wall temperature,
    interior untouched bit for bit, wall-row mass conserved."""
    g, prv, _ = pair(d2q37, 8, 10)
    fill_random(prv, d2q37, seed=3)
    p = tl.PhysicsParams(tau=1.0, Twall_top=0.6, Twall_bot=0.8)
    top_rows = slice(g.Hy + g.Ly - 3, g.Hy + g.Ly)
    mid_rows = slice(g.Hy + 3, g.Hy + g.Ly - 3)
    interior = prv.pops[:, g.phys_x, mid_rows].clone()
    mass_top = prv.pops[:, g.phys_x, top_rows].sum().item()
    tl.bc(prv, p, d2q37)
    top = prv.pops[:, g.phys_x, top_rows].contiguous()
    bot = prv.pops[:, g.phys_x, g.Hy:g.Hy + 3].contiguous()
    for block, Tw in ((top, 0.6), (bot, 0.8)):
        _, ux, uy, T = tl.moments(block, d2q37)
        assert ux.abs().max().item() < 1e-14 and uy.abs().max().item() < 1e-14
        assert (T - Tw).abs().max().item() < 1e-12
    assert torch.equal(prv.pops[:, g.phys_x, mid_rows], interior)
    assert top.sum().item() == pytest.approx(mass_top, rel=1e-13)


# ----------------------------------------------------------------- collide --

def test_collide_infinite_tau_limit(d2q9):
    """test_kernels.py:264-269."""
    f = 0.2 + np.random.default_rng(13).random((9, 4))
    out = tl.collide(f, tl.PhysicsParams(tau=1e12), d2q9)
    assert np.allclose(out, f, rtol=1e-11)


# ------------------------------------------------------------------- fused --

def test_fused_matches_staged(d2q37):
    """test_kernels.py:287-299: fused == propagate then collide, bitwise."""
    p = tl.PhysicsParams(tau=0.8, gy=-1e-4)
    g, prv, nxt = pair(d2q37)
    fill_random(prv, d2q37, seed=23)
    periodic_fill(prv.pops)
    xs, ys = slice(g.Hx + 1, g.Hx + 7), slice(g.Hy + 2, g.Hy + 6)
    ref = tl.PopulationField(g, "nxt")
    tl.propagate(prv, ref, d2q37, (xs, ys))
    ref.pops[:, xs, ys] = tl.collide(ref.pops[:, xs, ys].contiguous(), p, d2q37)
    tl.propagate_collide_fused(prv, nxt, p, d2q37, (xs, ys))
    assert torch.equal(nxt.pops[:, xs, ys], ref.pops[:, xs, ys])


def test_fused_empty_region_is_noop(d2q9):
    """test_kernels.py:302-308: a zero-width region writes nothing."""
    g, prv, nxt = pair(d2q9)
    nxt.pops.fill_(0.25)
    empty = (slice(g.Hx, g.Hx), g.phys_y)
    tl.propagate_collide_fused(prv, nxt, tl.PhysicsParams(tau=0.8), d2q9, empty)
    assert bool((nxt.pops == 0.25).all())


def test_fused_single_site(d2q9):
    """test_kernels.py:311-321: one site = gather of its 9 upstream values,
    then collide."""
    p = tl.PhysicsParams(tau=0.8)
    g, prv, nxt = pair(d2q9)
    fill_random(prv, d2q9, seed=29)
    x, y = g.Hx + 2, g.Hy + 2
    tl.propagate_collide_fused(prv, nxt, p, d2q9, (slice(x, x + 1), slice(y, y + 1)))
    src = prv.numpy()
    gathered = np.array([src[l, x - d2q9.c[l, 0], y - d2q9.c[l, 1]] for l in range(9)])
    want = tl.collide(gathered[:, None], p, d2q9)
    assert np.array_equal(nxt.numpy()[:, x, y], want[:, 0])


def test_fused_rejects_bc_rows(d2q37):
    """test_kernels.py:324-329."""
    g, prv, nxt = pair(d2q37)
    with pytest.raises(tl.ContractViolation):
        tl.propagate_collide_fused(prv, nxt, tl.PhysicsParams(tau=0.8), d2q37,
                                   (g.phys_x, g.phys_y), exclude_y=[(g.Hy, g.Hy + 3)])
