"""The reference's host-side tests, one for one, on the drop-in package
(no GPU needed): tests/test_velocity_set.py, the host parts of
tests/test_geometry.py and tests/test_runtime.py, and acceptance criteria
c01, c06 and c07 of tests/test_acceptance.py.

Names, inputs and tolerances follow the reference test each one cites;
device-side tests of the same files are in tests/test_gpu_reference_*.py.
"""

import itertools
import math

import numpy as np
import pytest

import paper_1703_00185_b200 as tl
from paper_1703_00185_b200.planner import factor_pairs
from paper_1703_00185_b200.velocity_set import gaussian_moment


@pytest.fixture(scope="module")
def d2q37():
    return tl.build_velocity_set("D2Q37")


@pytest.fixture(scope="module")
def d2q9():
    return tl.build_velocity_set("D2Q9")


def wmoment(vs, a, b):
    """sum_l w_l cx^a cy^b."""
    c = vs.c.astype(float)
    return float(vs.w @ (c[:, 0] ** a * c[:, 1] ** b))


# ----------------------------------------------------- test_velocity_set.py --

def test_d2q37_counts(d2q37):
    """test_velocity_set.py:14-17."""
    assert (d2q37.Q, d2q37.max_hop) == (37, 3)
    assert len(set(map(tuple, d2q37.c.tolist()))) == 37


def test_d2q9_basics(d2q9):
    """test_velocity_set.py:20-26."""
    assert (d2q9.Q, d2q9.max_hop) == (9, 1)
    assert tuple(d2q9.c[0]) == (0, 0)
    assert abs(d2q9.w.sum() - 1.0) < 1e-15
    assert d2q9.cs2 == pytest.approx(1 / 3)


@pytest.mark.parametrize("name", ["D2Q37", "D2Q9"])
def test_closed_under_negation(name):
    """test_velocity_set.py:29-34."""
    vecs = set(map(tuple, tl.build_velocity_set(name).c.tolist()))
    assert {(-a, -b) for a, b in vecs} == vecs


@pytest.mark.parametrize("name", ["D2Q37", "D2Q9"])
def test_weights_positive_and_normalized(name):
    """test_velocity_set.py:37-40."""
    w = tl.build_velocity_set(name).w
    assert (w > 0).all() and abs(w.sum() - 1.0) < 1e-14


def test_d2q37_odd_moments_vanish(d2q37):
    """test_velocity_set.py:43-47: every moment of total order < 6 with an
    odd exponent vanishes."""
    for a, b in itertools.product(range(6), repeat=2):
        if a + b < 6 and (a % 2 or b % 2):
            assert abs(wmoment(d2q37, a, b)) < 1e-12, (a, b)


def test_d2q37_even_moments_gaussian(d2q37):
    """test_velocity_set.py:50-55: even moments through order 8 are those of
    the Gaussian with variance cs2."""
    for a, b in itertools.product(range(0, 9, 2), repeat=2):
        if a + b <= 8:
            assert abs(wmoment(d2q37, a, b) - gaussian_moment(a, b, d2q37.cs2)) < 1e-12


def test_d2q37_isotropic_fourth_moment(d2q37):
    """test_velocity_set.py:58-60."""
    assert wmoment(d2q37, 2, 2) == pytest.approx(d2q37.cs2 ** 2, abs=1e-13)


def test_d2q9_second_moment(d2q9):
    """test_velocity_set.py:63-65."""
    assert wmoment(d2q9, 2, 0) == pytest.approx(d2q9.cs2, abs=1e-15)
    assert wmoment(d2q9, 3, 1) == pytest.approx(0.0, abs=1e-15)


def test_unknown_name_rejected():
    """test_velocity_set.py:68-70."""
    with pytest.raises(tl.ConfigurationError):
        tl.build_velocity_set("D3Q19")


def test_velocity_lookup(d2q37):
    """test_velocity_set.py:73-77."""
    assert tuple(d2q37.c[d2q37.find(3, 1)]) == (3, 1)
    with pytest.raises(tl.ConfigurationError):
        d2q37.find(4, 0)


# -------------------------------------------- test_geometry.py (host part) --

def test_table2_lattice_extents(d2q37):
    """test_geometry.py:19-22 (paper Table 2)."""
    g = tl.LatticeGeometry(1024, 8192, 3, 3, d2q37.Q)
    assert (g.NX, g.NY) == (1030, 8198)


def test_degenerate_extent_rejected():
    """test_geometry.py:25-27."""
    with pytest.raises(tl.AllocationError):
        tl.LatticeGeometry(0, 4, 3, 3, 9)


def test_thin_halo_rejected(d2q37):
    """test_geometry.py:30-33 (checked before any device allocation)."""
    with pytest.raises(tl.AllocationError):
        tl.allocate_field(tl.LatticeGeometry(8, 8, 1, 1, d2q37.Q), d2q37)


def test_site_index_soa():
    """test_geometry.py:42-46."""
    g = tl.LatticeGeometry(4, 4, 3, 3, 9, tl.SOA)
    assert [tl.site_index(g, *i) for i in ((0, 0, 0), (1, 0, 0), (0, 1, 0))] == \
        [0, g.NX * g.NY, g.NY]


def test_site_index_aos():
    """test_geometry.py:49-53."""
    g = tl.LatticeGeometry(4, 4, 3, 3, 9, tl.AOS)
    x, y = divmod(5, g.NY)
    assert tl.site_index(g, 2, x, y) == 5 * g.Q + 2


def test_site_index_bounds():
    """test_geometry.py:56-62."""
    g = tl.LatticeGeometry(4, 4, 3, 3, 9)
    for bad in ((9, 0, 0), (0, g.NX, 0)):
        with pytest.raises(tl.ContractViolation):
            tl.site_index(g, *bad)


# --------------------------------------------- test_runtime.py (host part) --

def test_decompose_2d_grid():
    """test_runtime.py:12-22."""
    tiles = tl.decompose(3600, 3600, 16, (4, 4))
    assert len(tiles) == 16 and all((t.Lx, t.Ly) == (900, 900) for t in tiles)
    t5 = tiles[5]
    assert t5.coords == (1, 1) and (t5.x0, t5.y0) == (900, 900)
    assert t5.neighbors == {"left": 4, "right": 6, "up": 9, "down": 1}
    assert not (t5.uppermost or t5.lowermost)
    assert tiles[0].lowermost and tiles[0].neighbors["down"] is None
    assert tiles[15].uppermost and tiles[15].neighbors["up"] is None


def test_decompose_1d_ring_grid():
    """test_runtime.py:25-31 (grid attribute; the rest is in test_host.py)."""
    assert [t.grid for t in tl.decompose(64, 32, 4, "1d")] == [(4, 1)] * 4


def test_decompose_periodic_y_ring():
    """test_runtime.py:34-38."""
    tiles = tl.decompose(16, 16, 4, (1, 4), periodic_y=True)
    assert tiles[0].neighbors["down"] == 3 and tiles[3].neighbors["up"] == 0
    assert not any(t.uppermost or t.lowermost for t in tiles)


def test_decompose_rejects_indivisible_2d():
    """test_runtime.py:41-45 (second case)."""
    with pytest.raises(tl.ConfigurationError):
        tl.decompose(100, 100, 4, (2, 3))


def test_face_plan_depth_counts_d2q37(d2q37):
    """test_runtime.py:50-55."""
    plans = tl.face_plans(d2q37)
    for key in itertools.product((0, 1), (1, -1)):
        assert [len(ls) for ls in plans[key]] == [15, 8, 3]
    assert tl.boundary_bytes_per_site(d2q37) == 208


def test_face_plan_depth_counts_d2q9(d2q9):
    """test_runtime.py:58-61."""
    assert [len(ls) for ls in tl.face_plans(d2q9)[(0, 1)]] == [3, 0, 0]
    assert tl.boundary_bytes_per_site(d2q9) == 24


def test_face_plan_membership(d2q37):
    """test_runtime.py:64-71: depth-d plan = exactly the populations with
    c_x >= d."""
    plans = tl.face_plans(d2q37)
    for d in (1, 2, 3):
        members = set(plans[(0, 1)][d - 1])
        assert members == {l for l in range(37) if d2q37.c[l, 0] >= d}


def test_fabric_roundtrip():
    """test_runtime.py:76-80."""
    fab = tl.Fabric(2, timeout=1.0)
    fab.send(0, 1, "x+", 7, np.arange(3.0))
    assert np.array_equal(fab.recv(1, 0, "x+", 7), np.arange(3.0))


def test_fabric_step_mismatch():
    """test_runtime.py:83-87."""
    fab = tl.Fabric(2, timeout=1.0)
    fab.send(0, 1, "x+", 3, None)
    with pytest.raises(tl.ProtocolError, match="expected step 4"):
        fab.recv(1, 0, "x+", 4)


def test_fabric_deadlock_names_rank():
    """test_runtime.py:90-93."""
    with pytest.raises(tl.DeadlockError, match="rank 1 stalled"):
        tl.Fabric(2, timeout=0.2).recv(1, 0, "x+", 0)


def test_deadlock_detection_surfaces():
    """test_runtime.py:291-296."""
    with pytest.raises(tl.DeadlockError) as err:
        tl.Fabric(3, timeout=0.15).recv(2, 1, "y+", 5)
    assert err.value.rank == 2


# ------------------------------------------ test_acceptance.py c01, c06, c07 --

def _gauss_1d(n, var):
    return 0.0 if n % 2 else math.prod(range(1, n, 2)) * var ** (n // 2)


def test_c01_weights_and_moments(d2q37):
    """test_acceptance.py:27-45: normalisation, parity to order 5, isotropy
    and Gaussian even moments to order 8, all within 1e-12."""
    assert abs(d2q37.w.sum() - 1.0) < 1e-12
    for a, b in itertools.product(range(6), repeat=2):
        if a + b <= 5 and (a % 2 or b % 2):
            assert abs(wmoment(d2q37, a, b)) < 1e-12
    for a, b in itertools.product(range(0, 9, 2), repeat=2):
        if a + b <= 8:
            m = wmoment(d2q37, a, b)
            assert abs(m - wmoment(d2q37, b, a)) < 1e-12
            assert abs(m - _gauss_1d(a, d2q37.cs2) * _gauss_1d(b, d2q37.cs2)) < 1e-12


def test_c06_planner_oracle():
    """test_acceptance.py:124-144: the integer grid equals brute force and
    the real optimum follows the closed form."""
    rng = np.random.default_rng(0)
    for _ in range(20):
        Lx, Ly = int(rng.integers(64, 4000)), int(rng.integers(64, 4000))
        Bx, By = float(rng.uniform(1e8, 1e10)), float(rng.uniform(1e8, 1e10))
        S = float(rng.uniform(8.0, 400.0))
        R = math.sqrt(Lx * By / (Ly * Bx))
        for Np in range(1, 65):
            real, best = tl.optimal_grid(tl.CostModelInput(Lx, Ly, Np, Bx, By, beta=1e-8, S=S))

            def cost(nx, ny):
                return S * (Ly / (By * ny) + Lx / (Bx * nx))

            assert cost(*best) == pytest.approx(min(cost(*g) for g in factor_pairs(Np)),
                                                rel=1e-13)
            assert real[0] == pytest.approx(math.sqrt(Np) * R, rel=1e-10)
            assert real[1] == pytest.approx(math.sqrt(Np) / R, rel=1e-10)


def test_c07_model_limits():
    """test_acceptance.py:147-161."""
    inp = tl.CostModelInput(4096, 4096, 8, Bx=1e30, By=1e30, beta=1e-8)
    assert abs(tl.predict_1d_overlap(inp).scale_violation - 1.0) < 1e-9
    with pytest.raises(tl.UnsupportedCaseError):
        tl.predict_2d_overlap(tl.CostModelInput(100, 200, 4, 1e9, 1e9, 1e-8))
    rng = np.random.default_rng(1)
    for _ in range(10):
        w = float(rng.uniform(1e-9, 1e-5))
        N, Np = int(rng.integers(1, 10 ** 7)), int(rng.integers(1, 4096))
        assert tl.brent_bound(w, N, Np) == w * (1.0 + (N - 1.0) / Np)
