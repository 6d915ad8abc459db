"""Host-side logic and the C ABI surface -- CPU only (no GPU needed)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

import paper_1703_00185_b200 as tl
from paper_1703_00185_b200 import _lib


# ---------------------------------------------------------- velocity set --

def test_velocity_set_matches_reference_bits(stencil):
    vs = tl.build_velocity_set("D2Q37")
    assert np.array_equal(vs.c, stencil["c"])
    assert np.array_equal(vs.w, stencil["w"])
    assert vs.cs2 == float(stencil["cs2"])
    assert vs.max_hop == 3 and vs.eq_order == 4


def test_velocity_set_invariants():
    vs = tl.build_velocity_set("D2Q37")
    c = vs.c.astype(float)
    assert abs(vs.w.sum() - 1.0) < 1e-12
    assert np.all(vs.w > 0)
    # closed under negation; partner of l within its shell is n-1-i
    for l in range(37):
        assert vs.find(-vs.c[l, 0], -vs.c[l, 1]) is not None
    assert abs(np.sum(vs.w * c[:, 0] * c[:, 0]) - vs.cs2) < 1e-12


def test_unknown_model():
    with pytest.raises(tl.ConfigurationError):
        tl.build_velocity_set("D3Q19")


# -------------------------------------------------------------- geometry --

def test_padding_and_extents():
    g = tl.LatticeGeometry(1024, 8192, 3, 3, 37)
    assert (g.NX, g.NY) == (1030, 8198)   # reference test_geometry.py:19-22
    assert g.phys_x == slice(3, 1027)


def test_site_index_layouts():
    g = tl.LatticeGeometry(4, 4, 3, 3, 9, tl.SOA)
    assert tl.site_index(g, 0, 0, 0) == 0
    assert tl.site_index(g, 1, 0, 0) == g.NX * g.NY
    assert tl.site_index(g, 0, 1, 0) == g.NY
    ga = tl.LatticeGeometry(4, 4, 3, 3, 9, tl.AOS)
    x, y = divmod(5, ga.NY)
    assert tl.site_index(ga, 2, x, y) == 5 * ga.Q + 2
    gc = tl.LatticeGeometry(4, 4, 3, 3, 9, tl.COLUMN)
    assert tl.site_index(gc, 0, 0, 1) == 1
    assert tl.site_index(gc, 1, 0, 0) == gc.NY
    assert tl.site_index(gc, 0, 1, 0) == gc.Q * gc.NY
    offs = {tl.site_index(gc, l, x, y) for l in range(9) for x in range(gc.NX)
            for y in range(gc.NY)}
    assert offs == set(range(9 * gc.NX * gc.NY))
    with pytest.raises(tl.ContractViolation):
        tl.site_index(g, 9, 0, 0)


def test_degenerate_geometry():
    with pytest.raises(tl.AllocationError):
        tl.LatticeGeometry(0, 4, 3, 3, 9)
    with pytest.raises(tl.AllocationError):
        tl.LatticeGeometry(4, 4, 3, 3, 9, "soa_bogus")


# --------------------------------------------------------------- runtime --

def test_decompose_1d_ring():
    tiles = tl.decompose(64, 32, 4, "1d")
    assert [t.x0 for t in tiles] == [0, 16, 32, 48]
    assert tiles[0].neighbors["left"] == 3 and tiles[3].neighbors["right"] == 0
    assert all(t.uppermost and t.lowermost for t in tiles)


def test_decompose_rejects_indivisible():
    with pytest.raises(tl.ConfigurationError, match="divides only by"):
        tl.decompose(100, 100, 3, "1d")


def test_face_plans_d2q37():
    vs = tl.build_velocity_set("D2Q37")
    plans = tl.face_plans(vs)
    for key in plans:
        assert [len(x) for x in plans[key]] == [15, 8, 3]
    assert list(plans[(0, 1)][2]) == [28, 35, 36]
    assert tl.boundary_bytes_per_site(vs) == 208


def test_fabric_protocol():
    fab = tl.Fabric(2, timeout=0.2)
    fab.send(0, 1, "x+", 3, "payload")
    with pytest.raises(tl.ProtocolError, match="expected step 4"):
        fab.recv(1, 0, "x+", 4)
    with pytest.raises(tl.DeadlockError, match="rank 1 stalled") as e:
        fab.recv(1, 0, "x+", 0)
    assert e.value.rank == 1
    fab.send(0, 1, "x-", 7, "ok")
    assert fab.recv(1, 0, "x-", 7) == "ok"


def test_simconfig_validation():
    with pytest.raises(tl.ConfigurationError):
        tl.SimConfig(Lx=8, Ly=8, schedule="bogus")
    with pytest.raises(tl.ConfigurationError):
        tl.SimConfig(Lx=8, Ly=8, walls=True, periodic_y=True)


def test_physics_params_validation():
    with pytest.raises(tl.DomainError):
        tl.PhysicsParams(tau=0.4)
    with pytest.raises(tl.DomainError):
        tl.PhysicsParams(tau=1.0, arith="bogus")


# ------------------------------------------------------------- the C ABI --

def _header_functions():
    src = open(os.path.join(ROOT, "include", "tlb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tlb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()          # loads without a GPU
    names = _header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    bound = {s[0] for s in _lib.SIGNATURES}
    assert set(names) == bound


def test_struct_layouts_match_header():
    assert ctypes.sizeof(_lib.TlbField) == 8 + 3 * 8 + 4 * 4
    assert ctypes.sizeof(_lib.TlbParams) == 6 * 8 + 2 * 4
    assert ctypes.sizeof(_lib.TlbStatus) == 48
    assert _lib.TlbStatus.negatives.offset == 40


def test_no_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(tl.DeviceError):
        tl.run(tl.SimConfig(Lx=8, Ly=8, steps=1))
    with pytest.raises(tl.DeviceError):
        tl.collide(np.ones((37, 2)), tl.PhysicsParams(tau=0.8),
                   tl.build_velocity_set("D2Q37"))
    lib = _lib.load()
    assert lib.tlb_device_count() == 0


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1703_00185_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in txt.replace("oracle/", "").lower() or \
                    "import oracle" not in txt, f
                assert "from oracle" not in txt and "import oracle" not in txt, f


# -------------------------------------------------------------------- io --

def test_macro_csv_matches_reference(tmp_path):
    from paper_1703_00185_b200 import io as tio
    g = golden("io.npz")
    m = g["macro_small"]
    tio.write_macro_csv(tmp_path / "m.csv", tl.MacroFields(*m))
    assert (tmp_path / "m.csv").read_text() == str(g["csv"])


def test_load_config(tmp_path):
    from paper_1703_00185_b200 import io as tio
    p = tmp_path / "c.yaml"
    p.write_text("Lx: 8\nLy: 4\n")
    assert tio.load_config(p) == {"Lx": 8, "Ly": 4}
    p.write_text("- 1\n- 2\n")
    with pytest.raises(tl.ConfigurationError):
        tio.load_config(p)
    with pytest.raises(tl.ConfigurationError):
        tio.load_config(tmp_path / "missing.yaml")


# --------------------------------------------------------------- planner --

def test_planner_matches_reference():
    from paper_1703_00185_b200 import planner as P
    g = golden("planner.npz")
    tab = P.BandwidthTable(g["tab_sizes"], g["tab_bw"])
    for row, want in zip(g["inputs"], g["outputs"]):
        Lx, Ly, Np, Bx, By, beta, S, use_tab = row
        Lx, Ly, Np = int(Lx), int(Ly), int(Np)
        inp = P.CostModelInput(Lx, Ly, Np, tab if use_tab else Bx, tab if use_tab else By,
                               beta, S)
        real, best = P.optimal_grid(inp)
        got = [P.predict_1d(inp).T_total, P.predict_2d(inp).T_total,
               P.predict_2d(inp, grid=best).T_total, P.predict_1d_overlap(inp).T_total,
               P.predict_1d_overlap(inp).scale_violation,
               P.predict_2d_overlap(inp).T_total if Lx == Ly else np.nan,
               P.comm_time_2d(inp, *best), real[0], real[1], best[0], best[1],
               P.surface_over_volume(Np, 2), P.brent_bound(beta, Lx * Ly, Np)]
        assert np.allclose(got, want, rtol=1e-12, atol=0, equal_nan=True), (row, got, want)


def test_planner_limits():
    from paper_1703_00185_b200 import planner as P
    inp = P.CostModelInput(4096, 4096, 8, Bx=1e30, By=1e30, beta=1e-8)
    assert abs(P.predict_1d_overlap(inp).scale_violation - 1.0) < 1e-9
    with pytest.raises(tl.UnsupportedCaseError):
        P.predict_2d_overlap(P.CostModelInput(100, 200, 4, 1e9, 1e9, 1e-8))
    with pytest.raises(tl.ContractViolation):
        P.CostModelInput(0, 10, 1, 1e9, 1e9, 1e-8)
    rows = P.scaling_curve(P.CostModelInput(512, 512, 1, 1e11, 1e11, 1e-10), [1, 2, 4])
    assert {r[1] for r in rows} == {"1d", "2d", "1d_overlap", "2d_overlap"}


def test_peer_neighbour_directions():
    """RankWorker._peer_neighbours: rank in each of the 8 peer directions
    (left, right, down, up, down-left, down-right, up-left, up-right),
    None where the side is self-periodic or a wall (csrc/tlb_peer.cuh)."""
    from types import SimpleNamespace
    from paper_1703_00185_b200.runtime import RankWorker

    def dirs(Lx, Ly, Np, tiling, periodic_y=False):
        out = []
        for t in tl.decompose(Lx, Ly, Np, tiling, periodic_y=periodic_y):
            nb = t.neighbors
            y_self = t.grid[1] == 1 and nb["up"] is not None
            w = SimpleNamespace(tile=t, x_self=nb["left"] == t.rank,
                                ex_up=nb["up"] is not None and not y_self,
                                ex_down=nb["down"] is not None and not y_self,
                                _PEER_DIRS=RankWorker._PEER_DIRS)
            out.append(RankWorker._peer_neighbours(w))
        return out

    # 1-D ring of 4 with walls: left/right only
    assert dirs(64, 16, 4, "1d")[1] == [0, 2, None, None, None, None, None, None]
    # 2x2 grid with walls: rank 0 (bottom-left) has right/up/up-right (= 1, 2, 3)
    # and, X being periodic, the same ranks on the left side
    d = dirs(32, 32, 4, (2, 2))
    assert d[0] == [1, 1, None, 2, None, None, 3, 3]
    assert d[3] == [2, 2, 1, None, 0, 0, None, None]
    # (1, 4) grid, periodic Y: X self-periodic -> only down/up
    d = dirs(16, 64, 4, (1, 4), periodic_y=True)
    assert d[0] == [None, None, 3, 1, None, None, None, None]
    # 3x3 periodic: all 8 distinct neighbours of the centre rank
    d = dirs(36, 36, 9, (3, 3), periodic_y=True)
    assert d[4] == [3, 5, 1, 7, 0, 2, 6, 8]
