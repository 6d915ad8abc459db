"""Multi-GPU paths (need >= 2 GPUs): one process per GPU over NCCL
(torchrun) and in-process ranks on several GPUs (peer copies)."""

import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("n", [2, 4])
def test_torchrun_nccl_ring_bitwise(n):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), os.path.join(ROOT, "tests", "dist_run.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0
    assert "DIST OK" in out.stdout


@pytest.mark.parametrize("mode", ["nccl", "p2p"])
def test_torchrun_stalled_neighbour_raises_deadlock(mode):
    """A rank whose ring neighbour stops stepping raises DeadlockError instead
    of hanging: NCCL ring -> host timeout + ring abort; peer stores -> the
    kernel's bounded wait flags PEER_TIMEOUT (tests/dist_stall.py)."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           "--nproc-per-node=2", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), os.path.join(ROOT, "tests", "dist_stall.py"), mode]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=180, cwd=ROOT)
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0
    assert "STALL OK" in out.stdout


def test_inprocess_ranks_on_two_gpus(orc):
    vs = tl.build_velocity_set("D2Q37")
    orc.set_stencil(vs.c, vs.w, vs.cs2)
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    res = tl.run(tl.SimConfig(Lx=64, Ly=32, Np=4, steps=6, params=p,
                              init="rayleigh-taylor", devices=(0, 1)))
    f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(64, 32, vs.cs2))
    want, _ = orc.run(f0, 6, orc.params6(0.8, 0.0, -1e-5, 1.0, p.Twall_top, p.Twall_bot))
    assert np.array_equal(res.populations, want)


@pytest.mark.parametrize("Np", [2, 4])
def test_inprocess_ring_pairs_on_two_gpus(orc, Np):
    """Two steps per launch across GPUs (tlb_peer_step2) with in-process
    ranks on two devices (Np=4: two ranks per device): bitwise vs the oracle,
    an odd step count (a final single step) included."""
    vs = tl.build_velocity_set("D2Q37")
    orc.set_stencil(vs.c, vs.w, vs.cs2)
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    Lx, Ly, steps = 24 * Np, 70, 9
    res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=Np, steps=steps, params=p,
                              init="rayleigh-taylor", devices=(0, 1), exchange="p2p",
                              temporal="on"))
    f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(Lx, Ly, vs.cs2))
    want, _ = orc.run(f0, steps, orc.params6(0.8, 0.0, -1e-5, 1.0, p.Twall_top, p.Twall_bot))
    assert np.array_equal(res.populations, want)


@pytest.mark.parametrize("temporal", ["on", "off"])
def test_inprocess_ring_of_eight_on_all_gpus(orc, temporal):
    """An 8-rank 1-D ring (the BASELINE's N=8 decomposition) spread over all
    visible GPUs (4 here: two ranks per device), peer stores from the step
    kernels, pairs and single steps: bitwise vs the oracle.  The closest this
    harness gets to 8 B200s -- every rank talks to its two neighbours only."""
    vs = tl.build_velocity_set("D2Q37")
    orc.set_stencil(vs.c, vs.w, vs.cs2)
    p = tl.PhysicsParams(tau=0.8, gy=-1e-5, Twall_top=0.9 * vs.cs2, Twall_bot=1.1 * vs.cs2)
    Lx, Ly, steps = 8 * 24, 70, 7
    res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=8, steps=steps, params=p,
                              init="rayleigh-taylor", exchange="p2p", temporal=temporal,
                              devices=tuple(range(torch.cuda.device_count()))))
    f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(Lx, Ly, vs.cs2))
    want, _ = orc.run(f0, steps, orc.params6(0.8, 0.0, -1e-5, 1.0, p.Twall_top, p.Twall_bot))
    assert np.array_equal(res.populations, want)


@pytest.mark.parametrize("n", [2, 4])
def test_torchrun_bench_config_pairs(n):
    """configs[2] at N = 2 / 4 (1920x2048 per GPU) under torchrun: exact pairs
    through the ring two-step kernel == exact single steps bitwise; the fast
    headline path within the 1e-12 contract (tests/dist_fullsize.py)."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr", "127.0.0.1",
           "--master-port", str(_port()), os.path.join(ROOT, "tests", "dist_fullsize.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(out.stdout[-3000:], out.stderr[-3000:])
    assert out.returncode == 0
    assert "FULLSIZE OK" in out.stdout
