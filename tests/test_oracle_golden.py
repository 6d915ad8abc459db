"""Pin the C oracle (oracle/tlb_oracle.c) to the REAL reference.

The fixtures in tests/golden/ were produced by the reference package itself
(tests/golden/make_golden.py); every comparison here is bitwise.  This is what
makes the oracle trustworthy as the checker for the CUDA path.
"""

import hashlib

import numpy as np
import pytest

from conftest import fingerprints, golden


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a, dtype=np.float64).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="module")
def kern():
    return golden("kernels.npz")


@pytest.fixture(scope="module")
def runs():
    return golden("runs.npz")


def test_propagate_bitwise(orc, kern):
    prv = kern["prv_0"].copy()
    nxt = np.zeros_like(prv)
    orc.propagate(prv, nxt, 3)
    assert np.array_equal(nxt, kern["prop_0"])


def test_bc_bitwise(orc, kern):
    f = kern["prop_0"].copy()
    orc.bc(f, 3, orc.params6(*kern["params"]))
    assert np.array_equal(f, kern["bc_0"])


@pytest.mark.parametrize("seed", [0, 23])
def test_collide_and_moments_bitwise(orc, kern, seed):
    prv = kern[f"prv_{seed}"].copy()
    nxt = np.zeros_like(prv)
    orc.propagate(prv, nxt, 3)
    blk = nxt[:, 3:19, 3:19]
    p6 = orc.params6(*kern["params"])
    assert np.array_equal(orc.collide(blk, p6), kern[f"collide_{seed}"])
    assert np.array_equal(np.stack(orc.moments(blk)), kern[f"mom_{seed}"])


def test_fused_bitwise(orc, kern):
    prv = kern["prv_0"].copy()
    out = np.zeros_like(prv)
    orc.fused(prv, out, 3, orc.params6(*kern["params"]), (4, 17, 6, 16))
    assert np.array_equal(out, kern["fused_0"])


@pytest.mark.parametrize("order", [2, 3, 4])
def test_equilibrium_bitwise(orc, kern, order):
    assert np.array_equal(orc.equilibrium(*kern["eq_in"], order=order),
                          kern[f"eq_out_{order}"])


def test_rest_equilibrium_is_w(orc, stencil):
    # reference tests/test_kernels.py:124-126
    f = orc.equilibrium(1.0, 0.0, 0.0, float(stencil["cs2"]))
    assert np.array_equal(f, stencil["w"])


def test_run_rt_walls_bitwise(orc, runs):
    out, neg = orc.run(runs["rt_f0"], 20, orc.params6(*runs["rt_params"]))
    assert np.array_equal(out, runs["rt_f20"])
    assert np.array_equal(neg, runs["rt_f20_negatives"])


def test_run_random_walls_bitwise(orc, runs):
    out, _ = orc.run(runs["rw_f0"], 6, orc.params6(*runs["rw_params"]))
    assert np.array_equal(out, runs["rw_f6"])


def test_run_periodic_bitwise(orc, runs):
    out, _ = orc.run(runs["pp_f0"], 10, orc.params6(*runs["pp_params"]),
                     ymode="periodic")
    assert np.array_equal(out, runs["pp_f10"])


def test_rt_init_macro_bitwise(orc, stencil):
    g = golden("rt_init.npz")
    rho, ux, uy, T = orc.rayleigh_taylor_macro(64, 32, float(stencil["cs2"]))
    assert np.array_equal(rho, g["rho"]) and np.array_equal(T, g["T"])
    assert sha16(orc.equilibrium(rho, ux, uy, T)) == str(g["f0_sha"])


def test_rt256_fingerprint_100_steps(orc, stencil, runs):
    """SURVEY §8c known answer: RT 256x128, 100 staged steps."""
    fp = fingerprints()
    assert sha16(stencil["w"]) == fp["w"]
    f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(256, 128, float(stencil["cs2"])))
    assert sha16(f0) == fp["rt256_f0"]
    out, neg = orc.run(f0, 100, orc.params6(*runs["rt_params"]))
    assert sha16(out) == fp["rt256_f100"]
    assert float(out.sum()) == fp["rt256_f100_sum"]


def test_degenerate_state_reported(orc):
    f = np.zeros((37, 4))
    with pytest.raises(orc.OracleError) as e:
        orc.moments(f)
    assert e.value.code == 1
