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
from .errors import ConfigurationError, ThermoLBError
from .geometry import MacroFields
from .init import initial_macro
from .kernels import PhysicsParams, equilibrium, moments
from .runtime import DEFAULT_HALO, DistFabric, Fabric, RankWorker, decompose
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


def _dist_rank_setup(cfg):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() == cfg.Np \
            and cfg.Np > 1:
        return dist
    return None


def run(cfg: SimConfig, f0=None) -> RunResult:
    """Execute cfg.steps time steps on cfg.Np ranks (sim.py:62-129).

    ``f0`` (optional, an extension): a (Q, Lx, Ly) initial state -- numpy, a
    (pinned) host tensor or a device tensor -- used instead of cfg.init."""
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
                           timing=cfg.timing)
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
        workers.append(w)

    snaps = {}
    if dist is not None:
        dist.barrier()
    t0 = time.perf_counter()
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
                snaps[s] = [(w.tile, w.physical_block())]
        for s in range(0 if not single else cfg.steps, cfg.steps):
            # lock step over the in-process ranks: every rank's sends are
            # posted before any rank waits (Y faces, then X faces)
            for phase in ("step_begin", "step_mid", "step_end"):
                for w in workers:
                    with torch.cuda.device(w.device):
                        getattr(w, phase)(s)
            if cfg.debug_poison:
                for w in workers:
                    if not bool(torch.isfinite(w.physical_block()).all()):
                        raise ThermoLBError(
                            f"rank {w.tile.rank}: NaN reached physical cells at step {s}")
            if cfg.snapshot_every and (s + 1) % cfg.snapshot_every == 0:
                snaps[s + 1] = [(w.tile, w.physical_block()) for w in workers]
        for w in workers:
            w.synchronize()
        wall = time.perf_counter() - t0
        for w in workers:
            w.collect()
    except ThermoLBError as exc:
        rank = getattr(exc, "rank", None)
        raise ThermoLBError(f"rank {rank if rank is not None else '?'} failed: {exc!r}") from exc

    def assemble(blocks):
        out = torch.empty((vs.Q, cfg.Lx, cfg.Ly), dtype=torch.float64,
                          device=workers[0].device)
        for tile, b in blocks:
            out[:, tile.x0:tile.x0 + tile.Lx, tile.y0:tile.y0 + tile.Ly].copy_(b)
        return out

    blocks = [(w.tile, w.physical_block()) for w in workers]
    metrics = []
    for w in workers:
        for s, row in enumerate(w.metrics):
            metrics.append({"step": s, "rank": w.tile.rank, **row})

    if dist is not None:
        # gather the tiles on rank 0 (NCCL gather over NVLink)
        mine = blocks[0][1]
        gathered = [torch.empty_like(mine) for _ in range(cfg.Np)] if rank == 0 else None
        dist.gather(mine, gathered, dst=0)
        dist.barrier()
        for w in workers:
            w.close()
        fabric.close()
        if rank != 0:
            mlups = cfg.Lx * cfg.Ly * cfg.steps / (wall * 1e6) if cfg.steps else 0.0
            return RunResult(None, None, metrics, mlups, wall, [])
        blocks = [(tiles[r], gathered[r]) for r in range(cfg.Np)]
        snaps = {}
    final = assemble(blocks)
    snap_list = [(s, _macro_of(assemble(b), vs, host)) for s, b in sorted(snaps.items())]
    macro = _macro_of(final, vs, host)
    if host:
        final = final.cpu().numpy()
    mlups = (cfg.Lx * cfg.Ly * cfg.steps / (wall * 1e6)) if cfg.steps else 0.0
    return RunResult(final, macro, metrics, mlups, wall, snap_list)
