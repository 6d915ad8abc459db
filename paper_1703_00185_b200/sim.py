"""Run orchestration (sim.py of the reference, sim.py:17-129) on B200s.

``run(SimConfig)`` keeps the reference's signature, result type and MLUPS
definition (Lx*Ly*steps / (wall*1e6), sim.py:127).  Ranks are either
in-process tiles (one process driving one or more GPUs; the reference's
"simulated ranks") or, when torch.distributed is initialised with
world_size == Np, one process per GPU exchanging X faces over NCCL.
"""

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigurationError, DegenerateStateError, ThermoLBError
from .geometry import MacroFields
from .init import initial_macro
from .kernels import PhysicsParams, equilibrium, field_desc, moments
from .runtime import (DEFAULT_HALO, DistFabric, Fabric, RankWorker, decompose,
                      link_local_peers)
from .velocity_set import build_velocity_set


@dataclass
class SimConfig:
    """Everything one run needs (sim.py:17-44).  Extra keys: ``devices`` (GPU
    indices for in-process ranks; default all visible, round-robin) and
    ``output`` ("host": numpy results like the reference; "device": torch
    CUDA tensors)."""

    Lx: int
    Ly: int
    model: str = "D2Q37"
    tiling: "str | tuple" = "1d"
    Np: int = 1
    schedule: str = "overlapped"
    steps: int = 0
    params: PhysicsParams = field(
        default_factory=lambda: PhysicsParams(tau=1.0, gx=0.0, gy=-1e-4))
    walls: bool = True
    periodic_y: bool = False
    layout: str = "column"   # storage order only; results are layout-independent
    halo: int = DEFAULT_HALO
    init: str = "uniform"
    init_kwargs: dict = field(default_factory=dict)
    snapshot_every: int = 0
    debug_poison: bool = False
    recv_timeout: float = 60.0
    devices: "tuple | None" = None
    output: str = "host"
    exchange: str = "auto"   # one process per GPU: "p2p" (NVLink peer stores fused into the
                             # step kernel) where it applies, else the "nccl" ring
    timing: str = "sampled"  # per-step device timers: "sampled" (1 in 32), "every", "off"
    temporal: str = "auto"   # two steps per launch on a single tile (csrc/tb2.cu): "auto"
                             # (fast arithmetic), "on" (also exact), "off"

    def __post_init__(self):
        if self.schedule not in ("staged", "overlapped"):
            raise ConfigurationError(f"unknown schedule {self.schedule!r}")
        if self.walls and self.periodic_y:
            raise ConfigurationError("walls and periodic_y are mutually exclusive")
        if self.output not in ("host", "device"):
            raise ConfigurationError(f"unknown output {self.output!r}")


@dataclass
class RunResult:
    populations: object      # (Q, Lx, Ly) final state (None on ranks != 0 under torchrun)
    macro: MacroFields
    metrics: list            # rows: dict per (step, rank)
    mlups: float
    wall_seconds: float
    snapshots: list          # (step, MacroFields)


def _macro_of(f, vs, host):
    rho, ux, uy, T = moments(f, vs)
    if host:
        rho, ux, uy, T = (a.cpu().numpy() for a in (rho, ux, uy, T))
    return MacroFields(rho, ux, uy, T)


def _tile_macro(w):
    """(4, Lx, Ly) device tensor of the tile's rho, ux, uy, T (moments,
    kernels.py:41-71, with its rho <= 0 check) straight from the field: no
    copy of the populations."""
    torch = _lib.torch_cuda()
    g = w.geom
    out = torch.empty((4, g.Lx, g.Ly), dtype=torch.float64, device=w.device)
    st = _lib.Status(w.device)
    with torch.cuda.stream(w.stream):
        st.buf.record_stream(w.stream)
        _lib.check(_lib.load().tlb_moments(
            field_desc(w.prv), _lib.region(g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly),
            *[out[k].data_ptr() for k in range(4)], g.Ly, 1, st.ptr,
            w.stream.cuda_stream), "moments")
    torch.cuda.current_stream(w.device).wait_stream(w.stream)
    if st.read().flags & _lib.ST_DEGENERATE:
        bad = torch.nonzero(~(out[0] > 0.0)).cpu().numpy()
        raise DegenerateStateError(f"rank {w.tile.rank}: non-positive density at "
                                   f"{bad[:5].tolist()}", sites=bad)
    return out


def _tile_pops(w):
    """The tile's physical populations as Q (Lx, Ly) device views (no copy)."""
    g = w.geom
    p = w.prv.pops
    return [p[l, g.phys_x, g.phys_y] for l in range(p.shape[0])]


def _dist_rank_setup(cfg):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() == cfg.Np \
            and cfg.Np > 1:
        return dist
    return None


class _Gather:
    """Tiles -> one (C, Lx, Ly) array: pinned host memory ('host' output) or a
    device tensor ('device').  Tiles travel one channel (population or
    macro field) at a time, so no full-tile copy is ever made; under
    torchrun the other ranks' channels arrive at rank 0 by NCCL
    point-to-point into one (Lx_tile, Ly_tile) staging buffer."""

    def __init__(self, cfg, tiles, host, device, dist=None):
        self.cfg, self.tiles, self.host, self.device, self.dist = cfg, tiles, host, device, dist

    def __call__(self, mine, rank=0):
        """mine: {rank: list of C (tx, ty) device tensors} of this process."""
        torch = _lib.torch_cuda()
        cfg, dist = self.cfg, self.dist
        chans = next(iter(mine.values()))
        C = len(chans)
        if dist is not None and rank != 0:
            for c in chans:
                dist.send(c.contiguous(), dst=0)
            return None
        shape = (C, cfg.Lx, cfg.Ly)
        if self.host:
            out = torch.empty(shape, dtype=torch.float64, pin_memory=True)
        else:
            out = torch.empty(shape, dtype=torch.float64, device=self.device)
        stage = None
        for t in self.tiles:
            dst = out[:, t.x0:t.x0 + t.Lx, t.y0:t.y0 + t.Ly]
            for c in range(C):
                if t.rank in mine:
                    dst[c].copy_(mine[t.rank][c])
                else:
                    if stage is None:
                        stage = torch.empty((t.Lx, t.Ly), dtype=torch.float64,
                                            device=self.device)
                    dist.recv(stage, src=t.rank)
                    dst[c].copy_(stage)
        return out.numpy() if self.host else out


def run(cfg: SimConfig, f0=None) -> RunResult:
    """Execute cfg.steps time steps on cfg.Np ranks (sim.py:62-129).

    ``f0`` (optional, an extension): a (Q, Lx, Ly) initial state -- numpy, a
    (pinned) host tensor or a device tensor -- used instead of cfg.init.

    Snapshots are reduced to (rho, u, T) on the device as they are taken
    (the reference keeps MacroFields, sim.py:89-90, 119-125), also with one
    process per GPU: the tiles' macro fields are gathered on rank 0."""
    torch = _lib.torch_cuda()
    vs = build_velocity_set(cfg.model)
    tiles = decompose(cfg.Lx, cfg.Ly, cfg.Np, cfg.tiling, periodic_y=cfg.periodic_y)
    macro0 = None
    if f0 is None:
        macro0 = initial_macro(cfg.init, cfg.Lx, cfg.Ly, vs, **cfg.init_kwargs)
    elif tuple(f0.shape) != (vs.Q, cfg.Lx, cfg.Ly):
        raise ConfigurationError(f"f0 has shape {tuple(f0.shape)}, expected "
                                 f"{(vs.Q, cfg.Lx, cfg.Ly)}")
    dist = _dist_rank_setup(cfg)
    host = cfg.output == "host"
    rank = 0

    if dist is not None:
        rank = dist.get_rank()
        dev = torch.device("cuda", torch.cuda.current_device())
        fabric = DistFabric(timeout=cfg.recv_timeout)
        my_tiles = [tiles[rank]]
        devices = [dev]
    else:
        fabric = Fabric(cfg.Np, timeout=cfg.recv_timeout)
        ndev = torch.cuda.device_count()
        idx = cfg.devices if cfg.devices else tuple(range(ndev))
        devices = [torch.device("cuda", idx[t.rank % len(idx)]) for t in tiles]
        my_tiles = tiles

    workers = []
    for i, tile in enumerate(my_tiles):
        dev = devices[i]
        with torch.cuda.device(dev):
            w = RankWorker(tile, vs, cfg.params, fabric, schedule=cfg.schedule,
                           walls=cfg.walls, layout=cfg.layout, halo=cfg.halo,
                           debug_poison=cfg.debug_poison, device=dev,
                           periodic_y=cfg.periodic_y, exchange=cfg.exchange,
                           timing=cfg.timing, temporal=cfg.temporal)
        workers.append(w)
    if dist is None and cfg.Np > 1 and cfg.exchange == "p2p":
        # in-process ranks with the peer-store step kernel of one process
        # per GPU (plain device pointers instead of CUDA IPC)
        link_local_peers(workers, strict=True)
    for w in workers:
        tile, dev = w.tile, w.device
        with torch.cuda.device(dev):
            sl = (slice(tile.x0, tile.x0 + tile.Lx), slice(tile.y0, tile.y0 + tile.Ly))
            if macro0 is not None:
                ts = [torch.as_tensor(np.ascontiguousarray(a[sl], dtype=np.float64),
                                      device=dev) for a in macro0]
                w.load_block(equilibrium(*ts, vs))
            else:
                src = f0[:, sl[0], sl[1]]
                if isinstance(src, np.ndarray):
                    src = torch.from_numpy(np.ascontiguousarray(src))
                w.load_block(src.to(dev, non_blocking=True))
            w.synchronize()

    gather = _Gather(cfg, tiles, host, workers[0].device, dist)
    snap_list = []

    def snapshot(step):
        mine = {}
        for w in workers:
            with torch.cuda.device(w.device):
                mine[w.tile.rank] = list(_tile_macro(w))
        m = gather(mine, rank)
        if m is not None:
            snap_list.append((step, MacroFields(*[m[k] for k in range(4)])))

    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
    err = None
    wall = 0.0
    try:
        single = (len(workers) == 1 and dist is None and not cfg.debug_poison
                  and workers[0].graphable())
        s = 0
        while single and s < cfg.steps:
            # one self-periodic tile: replayed CUDA graphs of the step sequence
            w = workers[0]
            n = cfg.steps - s
            if cfg.snapshot_every:
                n = min(n, cfg.snapshot_every - s % cfg.snapshot_every)
            with torch.cuda.device(w.device):
                w.run_steps(s, n)
            s += n
            if cfg.snapshot_every and s % cfg.snapshot_every == 0:
                snapshot(s)
        # ranks on a 1-D ring of peers pair steps (tlb_peer_step2) unless a
        # snapshot falls between the two
        pair = not single and all(w.pairable() for w in workers)
        s = 0 if not single else cfg.steps
        while s < cfg.steps:
            every = cfg.snapshot_every
            if pair and s + 1 < cfg.steps and not (every and (s + 1) % every == 0):
                for w in workers:
                    with torch.cuda.device(w.device):
                        w.prime_halos(s, 6)
                for w in workers:
                    with torch.cuda.device(w.device):
                        w.step_pair(s)
                s += 2
            else:
                for w in workers:
                    with torch.cuda.device(w.device):
                        w.prime_halos(s, 3)
                # lock step over the in-process ranks: every rank's sends are
                # posted before any rank waits (Y faces, then X faces)
                for phase in ("step_begin", "step_mid", "step_end"):
                    for w in workers:
                        with torch.cuda.device(w.device):
                            getattr(w, phase)(s)
                s += 1
            if cfg.debug_poison:
                for w in workers:
                    if not bool(torch.isfinite(w.physical_block()).all()):
                        raise ThermoLBError(
                            f"rank {w.tile.rank}: NaN reached physical cells at step {s - 1}")
            if every and s % every == 0:
                snapshot(s)
        for w in workers:
            w.synchronize()
        wall = time.perf_counter() - t0
        for w in workers:
            w.collect()
    except ThermoLBError as exc:
        err = exc
    if dist is not None:
        # every rank learns whether any rank failed before the collectives
        # below, so one rank's error is a clean error everywhere, not a hang
        flag = torch.tensor([1.0 if err is not None else 0.0], device=workers[0].device)
        dist.all_reduce(flag, op=dist.ReduceOp.MAX)
        if err is None and flag.item() > 0:
            err = ThermoLBError(f"rank {rank}: stopped because another rank failed")
    if err is not None:
        for w in workers:
            try:
                w.close()
            except ThermoLBError:
                pass
        if dist is not None:
            fabric.abort_ring()
            fabric.close()
        r = getattr(err, "rank", None)
        raise ThermoLBError(f"rank {r if r is not None else '?'} failed: {err!r}") from err

    metrics = []
    for w in workers:
        for s, row in enumerate(w.metrics):
            metrics.append({"step": s, "rank": w.tile.rank, **row})
    mlups = (cfg.Lx * cfg.Ly * cfg.steps / (wall * 1e6)) if cfg.steps else 0.0

    # final state and its macro fields: tile by tile into one array
    blocks, macros = {}, {}
    for w in workers:
        with torch.cuda.device(w.device):
            w.synchronize()
            blocks[w.tile.rank] = _tile_pops(w)
            macros[w.tile.rank] = list(_tile_macro(w))
    final = gather(blocks, rank)
    macro = gather(macros, rank)
    for w in workers:
        w.close()
    if dist is not None:
        dist.barrier()
        fabric.close()
        if rank != 0:
            return RunResult(None, None, metrics, mlups, wall, [])
    return RunResult(final, MacroFields(*[macro[k] for k in range(4)]), metrics, mlups,
                     wall, snap_list)
