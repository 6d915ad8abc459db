"""The peer-store step kernel (csrc/tlb_peer.cuh, the default halo exchange
of one process per GPU) driven by in-process ranks on ONE GPU.

link_local_peers hands every rank its neighbours' buffers and mailboxes as
plain device pointers, so the kernel that runs under torchrun -- border
blocks waiting on the neighbours' mailboxes, storing the face-plan lines
(runtime.py:94-107) into their halos, publishing each step with its tag --
runs here with no CUDA IPC and no second GPU.  Parity against the C oracle:
bitwise for the exact arithmetic, 1e-12 relative for fast; the rank layouts
of reference tests/test_acceptance.py:106-121 (rank invariance) and the
debug poisoning of runtime.py:288-294 / sim.py:84-88.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1703_00185_b200 as tl  # noqa: E402
from paper_1703_00185_b200 import _lib  # noqa: E402
from paper_1703_00185_b200.errors import (DeadlockError, ProtocolError,  # noqa: E402
                                          ThermoLBError)
from paper_1703_00185_b200.runtime import link_local_peers  # noqa: E402

VS = None


def _vs():
    global VS
    if VS is None:
        VS = tl.build_velocity_set("D2Q37")
    return VS


def _params(arith="exact"):
    vs = _vs()
    return tl.PhysicsParams(tau=0.8, gx=2e-6, gy=-1e-5, Twall_top=0.9 * vs.cs2,
                            Twall_bot=1.1 * vs.cs2, arith=arith)


def _oracle(orc, Lx, Ly, steps, p, periodic):
    vs = _vs()
    orc.set_stencil(vs.c, vs.w, vs.cs2)
    f0 = orc.equilibrium(*orc.rayleigh_taylor_macro(Lx, Ly, vs.cs2))
    want, neg = orc.run(f0, steps, orc.params6(p.tau, p.gx, p.gy, p.dt, p.Twall_top,
                                               p.Twall_bot),
                        ymode="periodic" if periodic else "walls")
    return want, neg


CASES = [
    # (Np, tiling, Lx, Ly, periodic_y)
    (2, "1d", 2 * 24, 40, False),       # 1-D ring, walls
    (4, "1d", 4 * 16, 36, False),       # 1-D ring of 4, walls
    (8, "1d", 8 * 12, 36, False),       # 1-D ring of 8
    (2, (1, 2), 40, 2 * 20, True),      # Y split only: X self-periodic, periodic Y ring
    (4, (1, 4), 36, 4 * 12, True),
    (4, (2, 2), 2 * 20, 2 * 18, False),  # 2-D with walls: corners go diagonal
    (4, (2, 2), 2 * 20, 2 * 18, True),   # 2-D, periodic Y: same rank above and below
]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"{c[0]}-{c[1]}-{c[4]}")
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_peer_step_matches_oracle(orc, case, arith):
    Np, tiling, Lx, Ly, periodic = case
    steps = 9
    p = _params(arith)
    res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=Np, tiling=tiling, steps=steps, params=p,
                              init="rayleigh-taylor", exchange="p2p", walls=not periodic,
                              periodic_y=periodic, devices=(0,)))
    want, neg = _oracle(orc, Lx, Ly, steps, p, periodic)
    if arith == "exact":
        assert np.array_equal(res.populations, want)
        # per-step negatives summed over ranks equal the oracle's
        got = np.zeros(steps, dtype=np.int64)
        for m in res.metrics:
            got[m["step"]] += m["negatives"]
        assert np.array_equal(got, np.asarray(neg)[:steps])
    else:
        assert np.max(np.abs(res.populations - want) / np.abs(want)) < 1e-12


def test_peer_step_is_the_kernel_used(orc):
    """The ranks really take the peer path (no Fabric payloads)."""
    vs = _vs()
    tiles = tl.decompose(48, 40, 2, "1d")
    fab = tl.Fabric(2)
    ws = [tl.RankWorker(t, vs, _params(), fab, schedule="overlapped", exchange="p2p",
                        device=torch.device("cuda", 0)) for t in tiles]
    assert link_local_peers(ws, strict=True)
    assert all(w.exchange_mode == "p2p" for w in ws)
    for w in ws:
        w.close()


def test_peer_step_debug_poison(orc):
    """NaN-poisoned halos never reach physical cells (reference
    runtime.py:288-294, tests/test_runtime.py:263-268): the peer kernel
    re-poisons prv's halos after its border blocks read them, so every halo
    value read later was stored by a neighbour in between."""
    p = _params()
    for Np, tiling, Lx, Ly, periodic in [(2, "1d", 48, 40, False), (4, (2, 2), 40, 36, True)]:
        res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=Np, tiling=tiling, steps=7, params=p,
                                  init="rayleigh-taylor", exchange="p2p",
                                  walls=not periodic, periodic_y=periodic,
                                  debug_poison=True, devices=(0,)))
        want, _ = _oracle(orc, Lx, Ly, 7, p, periodic)
        assert np.array_equal(res.populations, want)


def _linked_pair(timeout=60.0):
    vs = _vs()
    tiles = tl.decompose(48, 40, 2, "1d")
    fab = tl.Fabric(2, timeout=timeout)
    ws = [tl.RankWorker(t, vs, _params(), fab, schedule="overlapped", exchange="p2p",
                        device=torch.device("cuda", 0), timing="off") for t in tiles]
    link_local_peers(ws, strict=True)
    macro = tl.init.rayleigh_taylor_macro(48, 40, vs)
    for w in ws:
        t = w.tile
        sl = (slice(t.x0, t.x0 + t.Lx), slice(t.y0, t.y0 + t.Ly))
        w.load_block(tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(a[sl]),
                                                      device="cuda") for a in macro], vs))
    return ws


def test_peer_step_tag_mismatch_is_protocol_error():
    """Ranks stepping different step numbers: the step tags published with
    every step disagree -> ProtocolError (Fabric.recv, runtime.py:151-154),
    not a deadlock."""
    ws = _linked_pair()
    for s in range(3):
        for w in ws:
            w.step(s)
    ws[0].step(3)
    ws[1].step(4)      # rank 1 skipped a step number
    ws[0].step(4)
    ws[1].step(5)
    with pytest.raises(ProtocolError):
        for w in ws:
            w.collect()
    for w in ws:
        w.close()


def test_peer_step_stalled_neighbour_times_out():
    """A rank whose neighbour never steps raises DeadlockError after the
    fabric timeout (the kernel's bounded wait), and its own publication is
    poisoned so nobody consumes halos that were never written."""
    ws = _linked_pair(timeout=0.5)
    ws[0].step(0)
    ws[0].step(1)     # waits for rank 1's step 0, which never comes
    with pytest.raises(DeadlockError):
        ws[0].collect()
    mb = ws[1].mailbox.cpu().numpy().astype(np.uint64)
    assert mb[0] >> np.uint64(63) == 1           # rank 0's publication carries the failure
    ws[1].step(0)                                  # rank 1 sees the poisoned mailbox
    with pytest.raises((DeadlockError, ThermoLBError)):
        ws[1].step(1)
        ws[1].collect()
    for w in ws:
        w.close()


def test_peer_prime_then_reload(orc):
    """load_block re-primes the halos (tlb_peer_prime) and the step numbers
    may jump there; the state stays bitwise equal to the oracle."""
    ws = _linked_pair()
    vs = _vs()
    p = _params()
    for s in range(4):
        for w in ws:
            w.step(s)
    macro = tl.init.rayleigh_taylor_macro(48, 40, vs)
    for w in ws:
        t = w.tile
        sl = (slice(t.x0, t.x0 + t.Lx), slice(t.y0, t.y0 + t.Ly))
        w.load_block(tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(a[sl]),
                                                      device="cuda") for a in macro], vs))
    for s in range(100, 105):
        for w in ws:
            w.step(s)
    got = np.concatenate([w.physical_block().cpu().numpy() for w in ws], axis=1)
    for w in ws:
        w.collect()
        w.close()
    want, _ = _oracle(orc, 48, 40, 5, p, False)
    assert np.array_equal(got, want)


# ---- two steps per launch across the ring (tlb_peer_step2) ---------------

PAIR_CASES = [
    # (Np, Lx, Ly, periodic_y, steps, snapshot_every)
    (2, 2 * 40, 70, False, 8, 0),       # walls, several strips, even steps
    (2, 2 * 24, 40, True, 9, 0),        # periodic Y, odd: a final single step
    (4, 4 * 20, 130, False, 11, 3),     # 4 ranks, snapshots between pairs
    (3, 3 * 12, 24, False, 6, 0),       # the narrowest tile (12 columns)
    (8, 8 * 16, 40, False, 6, 0),       # a ring of 8 (the BASELINE's N=8) on one GPU
]


@pytest.mark.parametrize("case", PAIR_CASES, ids=lambda c: "-".join(map(str, c)))
@pytest.mark.parametrize("arith", ["exact", "fast"])
def test_peer_pairs_match_oracle(orc, case, arith):
    """In-process ranks on one GPU with temporal="on": the ring kernel's
    border runs read 6-column halos their neighbours stored and store their
    own; bitwise (exact) / 1e-12 (fast) against the oracle, per-step
    negatives, snapshots taken between pairs."""
    Np, Lx, Ly, periodic, steps, every = case
    p = _params(arith)
    res = tl.run(tl.SimConfig(Lx=Lx, Ly=Ly, Np=Np, tiling="1d", steps=steps, params=p,
                              init="rayleigh-taylor", exchange="p2p", walls=not periodic,
                              periodic_y=periodic, devices=(0,), temporal="on",
                              snapshot_every=every))
    want, neg = _oracle(orc, Lx, Ly, steps, p, periodic)
    if arith == "exact":
        assert np.array_equal(res.populations, want)
        got = np.zeros(steps, dtype=np.int64)
        for m in res.metrics:
            got[m["step"]] += m["negatives"]
        assert np.array_equal(got, np.asarray(neg)[:steps])
    else:
        assert np.max(np.abs(res.populations - want) / np.abs(want)) < 1e-12
    if every:
        assert [s for s, _ in res.snapshots] == list(range(every, steps + 1, every))


@pytest.mark.parametrize("order", [0, 1])
def test_peer_pairs_work_orders(orc, order):
    """The ring two-step kernel with both work orders (interior runs
    strip-major / run-major) and short runs: bitwise vs the oracle."""
    import ctypes
    lib = _lib.load()
    saved = []
    for key in (3, 4):
        v = ctypes.c_int(0)
        _lib.check(lib.tlb_get_tuning(key, ctypes.byref(v)), "get")
        saved.append((key, v.value))
    try:
        _lib.check(lib.tlb_set_tuning(4, order), "order")
        _lib.check(lib.tlb_set_tuning(3, 12), "run")
        p = _params()
        res = tl.run(tl.SimConfig(Lx=2 * 60, Ly=130, Np=2, tiling="1d", steps=6, params=p,
                                  init="rayleigh-taylor", exchange="p2p", devices=(0,),
                                  temporal="on"))
        want, _ = _oracle(orc, 120, 130, 6, p, False)
        assert np.array_equal(res.populations, want)
    finally:
        for key, v in saved:
            _lib.check(lib.tlb_set_tuning(key, v), "restore")


def test_peer_pairs_are_the_kernel_used():
    """temporal="on" ranks on a 1-D ring allocate 6 halo columns and pair."""
    vs = _vs()
    tiles = tl.decompose(48, 40, 2, "1d")
    fab = tl.Fabric(2)
    ws = [tl.RankWorker(t, vs, _params(), fab, schedule="overlapped", exchange="p2p",
                        device=torch.device("cuda", 0), temporal="on") for t in tiles]
    assert link_local_peers(ws, strict=True)
    assert all(w.geom.Hx == 6 and w.pairable() for w in ws)
    for w in ws:
        w.close()


def test_peer_pairs_mixed_with_single_steps(orc):
    """Pairs, then single steps, then pairs again (the halos are re-primed
    to 6 columns), then a reload: bitwise equal to the oracle."""
    vs = _vs()
    p = _params()
    tiles = tl.decompose(48, 40, 2, "1d")
    fab = tl.Fabric(2)
    ws = [tl.RankWorker(t, vs, p, fab, schedule="overlapped", exchange="p2p",
                        device=torch.device("cuda", 0), temporal="on") for t in tiles]
    link_local_peers(ws, strict=True)
    macro = tl.init.rayleigh_taylor_macro(48, 40, vs)
    for w in ws:
        t = w.tile
        sl = (slice(t.x0, t.x0 + t.Lx), slice(t.y0, t.y0 + t.Ly))
        w.load_block(tl.equilibrium(*[torch.as_tensor(np.ascontiguousarray(a[sl]),
                                                      device="cuda") for a in macro], vs))
    plan = ["pair", "single", "single", "pair", "pair", "single", "pair"]
    s = 0
    for kind in plan:
        for w in ws:
            (w.step_pair if kind == "pair" else w.step)(s)
        s += 2 if kind == "pair" else 1
    got = np.concatenate([w.physical_block().cpu().numpy() for w in ws], axis=1)
    for w in ws:
        w.collect()
        w.close()
    want, _ = _oracle(orc, 48, 40, s, p, False)
    assert np.array_equal(got, want)


def test_peer_pairs_stalled_neighbour_times_out():
    """A pair launch whose neighbour never steps: DeadlockError after the
    fabric timeout, no hang."""
    vs = _vs()
    tiles = tl.decompose(48, 40, 2, "1d")
    fab = tl.Fabric(2, timeout=0.5)
    ws = [tl.RankWorker(t, vs, _params(), fab, schedule="overlapped", exchange="p2p",
                        device=torch.device("cuda", 0), temporal="on", timing="off")
          for t in tiles]
    link_local_peers(ws, strict=True)
    for w in ws:
        w.load_block(torch.full((37, w.tile.Lx, 40), 0.02, dtype=torch.float64))
    ws[0].step_pair(0)      # primes (waits for rank 1's prime: never comes)
    with pytest.raises(DeadlockError):
        ws[0].collect()
    for w in ws:
        w.close()


@pytest.mark.parametrize("exchange", ["p2p", "auto"])
def test_six_wide_halos(orc, exchange):
    """The halo width is a parameter: 6-wide halos (what a ring rank that
    pairs steps allocates) with single steps through the peer kernel and
    through the in-process Fabric exchange: bitwise vs the oracle."""
    p = _params()
    res = tl.run(tl.SimConfig(Lx=48, Ly=40, Np=2, tiling="1d", steps=7, params=p,
                              init="rayleigh-taylor", exchange=exchange, devices=(0,),
                              halo=6, temporal="off"))
    want, _ = _oracle(orc, 48, 40, 7, p, False)
    assert np.array_equal(res.populations, want)
