"""Shared fixtures.  `gpu`-marked tests need a B200 (run through gpurun);
everything else runs on the CPU-only build container."""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: longer CPU test")


def golden(name):
    return np.load(os.path.join(GOLDEN, name))


def fingerprints():
    with open(os.path.join(GOLDEN, "fingerprints.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def stencil():
    return golden("stencil.npz")


@pytest.fixture(scope="session")
def orc(stencil):
    from oracle import oracle as O
    O.set_stencil(stencil["c"], stencil["w"], float(stencil["cs2"]))
    return O


def periodic_fill(pops, H=3):
    """Fill the H-wide halo frame of a (Q, NX, NY) array (numpy or torch)
    from the opposite physical edges, corners included -- the periodic
    wrap of the reference's tests/conftest.py:17-27.  X first, then Y over
    full columns, so corners come out right."""
    NX, NY = pops.shape[1], pops.shape[2]
    for axis, n in ((1, NX), (2, NY)):
        L = n - 2 * H
        lo_halo, hi_src = slice(0, H), slice(L, L + H)
        hi_halo, lo_src = slice(H + L, n), slice(H, 2 * H)
        for dst, src in ((lo_halo, hi_src), (hi_halo, lo_src)):
            idx_d = [slice(None)] * 3
            idx_s = [slice(None)] * 3
            idx_d[axis], idx_s[axis] = dst, src
            pops[tuple(idx_d)] = pops[tuple(idx_s)]


def random_state(NX, NY, seed=0, lo=0.5, Q=37):
    """lo + U[0, 1) of shape (Q, NX, NY): the same draws as the reference's
    tests/conftest.py:30-32 for a given seed."""
    return lo + np.random.default_rng(seed).random((Q, NX, NY))
