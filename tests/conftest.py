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
    """Wrap halos periodically in both directions (reference
    tests/conftest.py:17-27), on a (Q, NX, NY) array (numpy or torch)."""
    Q, NX, NY = pops.shape
    Lx, Ly = NX - 2 * H, NY - 2 * H
    pops[:, :H, :] = pops[:, Lx:Lx + H, :]
    pops[:, H + Lx:, :] = pops[:, H:2 * H, :]
    pops[:, :, :H] = pops[:, :, Ly:Ly + H]
    pops[:, :, H + Ly:] = pops[:, :, H:2 * H]


def random_state(NX, NY, seed=0, lo=0.5, Q=37):
    """Reference tests/conftest.py:30-32."""
    rng = np.random.default_rng(seed)
    return lo + rng.random((Q, NX, NY))
