"""Rank runtime on B200s: tiles, X-halo exchange, step schedules.

Mirrors runtime.py of the reference (/root/reference/pkg/src/thermolb/
runtime.py) for the 1-D X ring the north star names: ``decompose``,
``face_plans``, ``TileAssignment`` and ``RankWorker`` keep their names and
meaning.  What changes is the machinery under them:

* a rank owns a tile in HBM (one GPU per rank in production; several tiles
  may share a GPU for testing) and every per-step operation is a libtlb.so
  kernel launched on the rank's CUDA stream -- nothing is synchronous;
* the Fabric's queues become either ``Fabric`` (in-process ranks: device
  payload tensors handed over with a CUDA event, copied peer-to-peer when the
  ranks sit on different GPUs) or ``DistFabric`` (one process per GPU,
  torch.distributed point-to-point over NCCL/NVLink; gloo for the CPU tests);
* schedule "staged" is the reference's split path, op for op (extend walls,
  pbc_nc, pbc_c, propagate, bc, collide) -- bitwise the reference, 1184 B/site;
  schedule "overlapped" is the B200 path: one fused propagate+bc+collide
  kernel per region with the wall extension and the periodic wraps of a rank
  that is its own neighbour folded into its loads, the face exchanges (Y
  first, then X over the full height) on a high-priority side stream
  overlapped with the bulk, then the frame bands -- 592 B/site.

Both decompositions of the reference are supported: the 1-D X ring (the
north star) and the 2-D grid (Y chain with walls or Y ring).
"""

import collections
import queue
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import (ConfigurationError, DeadlockError, DegenerateStateError,
                     DeviceError, DomainError, ProtocolError, ThermoLBError)
from .geometry import LatticeGeometry, allocate_field, swap_buffers
from .kernels import WALL_ROWS, field_desc
from .velocity_set import VelocitySet

DEFAULT_HALO = 3
_POLL = 0.05


@dataclass
class TileAssignment:
    """One rank's tile: extents, grid coordinates and neighbour table
    (runtime.py:33-46)."""

    rank: int
    grid: tuple
    coords: tuple
    Lx: int
    Ly: int
    x0: int
    y0: int
    neighbors: dict
    uppermost: bool = False
    lowermost: bool = False


def _divisor_hint(L, axis):
    divs = [d for d in range(1, min(L, 64) + 1) if L % d == 0]
    return f"{axis} extent {L} divides only by {divs}"


def decompose(Lx, Ly, Np, tiling, periodic_y=False):
    """Uniform tiles of an (Lx, Ly) lattice on an nx x ny rank grid, ranks
    numbered row-major (x fastest); "1d" is the X ring (nx = Np).  Same
    tiles, neighbour table and errors as the reference (runtime.py:54-91):
    X always wraps; Y wraps only with periodic_y, else the bottom / top row
    of ranks owns the walls."""
    nx, ny = (Np, 1) if tiling == "1d" else tuple(tiling)
    if nx * ny != Np:
        raise ConfigurationError(f"grid {nx}x{ny} does not match Np={Np}")
    for L, n, ax in ((Lx, nx, "X"), (Ly, ny, "Y")):
        if L % n:
            name = "Lx" if ax == "X" else "Ly"
            raise ConfigurationError(f"{name}={L} not divisible by n{ax.lower()}={n}; "
                                     + _divisor_hint(L, ax))
    tx, ty = Lx // nx, Ly // ny

    def rank_of(ix, iy):
        return (iy % ny) * nx + ix % nx

    def tile(ix, iy):
        top, bottom = iy == ny - 1, iy == 0
        if periodic_y:
            up, down = rank_of(ix, iy + 1), rank_of(ix, iy - 1)
        else:
            up = None if top else rank_of(ix, iy + 1)
            down = None if bottom else rank_of(ix, iy - 1)
        return TileAssignment(
            rank=rank_of(ix, iy), grid=(nx, ny), coords=(ix, iy), Lx=tx, Ly=ty,
            x0=ix * tx, y0=iy * ty,
            neighbors={"left": rank_of(ix - 1, iy), "right": rank_of(ix + 1, iy),
                       "up": up, "down": down},
            uppermost=top and not periodic_y, lowermost=bottom and not periodic_y)

    return [tile(ix, iy) for iy in range(ny) for ix in range(nx)]


def face_plans(vs: VelocitySet, depth=DEFAULT_HALO):
    """For each face (axis, sign) and halo depth d = 1..depth, the
    populations that cross it that far: sign * c_l[axis] >= d
    (runtime.py:94-107).  plans[(axis, sign)][d - 1] -> index array."""
    c = np.asarray(vs.c)
    return {(axis, sign): [np.flatnonzero(sign * c[:, axis] >= d) for d in range(1, depth + 1)]
            for axis in (0, 1) for sign in (1, -1)}


def boundary_bytes_per_site(vs: VelocitySet, depth=DEFAULT_HALO):
    """The model's S (runtime.py:110-113): float64 values one boundary site
    sends across a face, over all depths."""
    return 8 * int(sum(ls.size for ls in face_plans(vs, depth)[(0, 1)]))


# --------------------------------------------------------------- fabrics --

class Fabric:
    """In-process point-to-point channels with the reference's semantics
    (runtime.py:116-160): FIFO per (src, dst, tag), every message carries its
    step; recv gives up after `timeout` seconds with DeadlockError naming the
    waiting rank, a message from another step is a ProtocolError, and one
    rank's failure (fail) makes every waiting recv abort.  Payloads are
    device tensors; the sender may attach a CUDA event so the receiver's
    stream waits for the pack without a host sync."""

    def __init__(self, Np, timeout=60.0):
        self.Np, self.timeout = Np, timeout
        self.channels = collections.defaultdict(queue.Queue)
        self.abort = threading.Event()
        self.failures = []
        self._lock = threading.Lock()

    def _chan(self, src, dst, tag):
        with self._lock:                     # defaultdict insertion is not atomic
            return self.channels[(src, dst, tag)]

    def send(self, src, dst, tag, step, payload, event=None):
        self._chan(src, dst, tag).put((step, payload, event))

    def recv(self, dst, src, tag, step, with_event=False):
        chan = self._chan(src, dst, tag)
        give_up = time.monotonic() + self.timeout
        msg = None
        while msg is None:
            if self.abort.is_set():
                raise ThermoLBError(f"rank {dst}: aborted by peer failure")
            try:
                msg = chan.get(timeout=min(_POLL, self.timeout))
            except queue.Empty:
                if time.monotonic() > give_up:
                    raise DeadlockError(f"rank {dst} stalled waiting for rank {src} "
                                        f"(tag {tag}, step {step})", rank=dst)
        got, payload, event = msg
        if got != step:
            raise ProtocolError(f"rank {dst}: expected step {step} from {src}/{tag}, got {got}")
        return (payload, event) if with_event else payload

    def fail(self, rank, exc):
        with self._lock:
            self.failures.append((rank, exc))
        self.abort.set()

    # -- face exchange used by RankWorker ---------------------------------
    # axis "x": +face -> right ("x+"), -face -> left ("x-"); received +face
    # comes from the left.  axis "y": +face -> up ("y+"), -face -> down
    # ("y-"); received +face comes from below.  Wall sides (no neighbour)
    # send and receive nothing (runtime.py:248-284).
    @staticmethod
    def _peers(w, axis):
        nb = w.tile.neighbors
        return (nb["right"], nb["left"]) if axis == "x" else (nb["up"], nb["down"])

    def start_face(self, w, step, axis, out_plus, out_minus):
        torch = _lib.torch_cuda()
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(w.device))
        fwd, bwd = self._peers(w, axis)
        if fwd is not None:
            self.send(w.tile.rank, fwd, axis + "+", step, out_plus, ev)
        if bwd is not None:
            self.send(w.tile.rank, bwd, axis + "-", step, out_minus, ev)
        return step

    def finish_face(self, w, handle, axis, in_plus, in_minus, stream=None):
        torch = _lib.torch_cuda()
        stream = stream or w.stream
        step = handle
        fwd, bwd = self._peers(w, axis)
        got = []
        for tag, src, dst in ((axis + "+", bwd, in_plus), (axis + "-", fwd, in_minus)):
            if src is None:
                got.append(False)
                continue
            payload, ev = self.recv(w.tile.rank, src, tag, step, with_event=True)
            if payload.numel() != dst.numel():
                raise ProtocolError(f"rank {w.tile.rank}: {axis.upper()} payload size mismatch")
            if ev is not None:
                stream.wait_event(ev)
            with torch.cuda.stream(stream):
                dst.copy_(payload, non_blocking=True)
            if payload.device == dst.device:
                payload.record_stream(stream)
            else:
                w.retain(payload)  # peer copy: keep alive until the next sync
            got.append(True)
        return got

    def start_x(self, w, step, out_plus, out_minus):
        return self.start_face(w, step, "x", out_plus, out_minus)

    def finish_x(self, w, handle, in_plus, in_minus, stream=None):
        return self.finish_face(w, handle, "x", in_plus, in_minus, stream)


class DistFabric:
    """X-face exchange between processes (one per GPU).

    With an NCCL process group the exchange is native: ``ring()`` builds a
    libtlb ``TlbRing`` (its own NCCL communicator over NVLink, unique id
    broadcast through torch.distributed) and RankWorker enqueues whole steps
    through ``tlb_ring_step`` -- pack, grouped send/recv on a high-priority
    side stream, bulk kernel, unpack and border kernel in one C call.
    ``start_x``/``finish_x`` (torch.distributed batched point-to-point) carry
    the same payloads for other backends; the CPU tests run them over gloo."""

    def __init__(self, group=None, timeout=60.0):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.timeout = timeout
        self.Np = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.abort = threading.Event()
        self.failures = []
        self._ring = None

    @property
    def native(self):
        return self.dist.get_backend(self.group) == "nccl"

    def ring(self, device_index):
        """The libtlb NCCL ring for this process (created on first use)."""
        if self._ring is None:
            import ctypes
            lib = _lib.load()
            uid = ctypes.create_string_buffer(128)
            if self.rank == 0:
                _lib.check(lib.tlb_nccl_unique_id(uid), "nccl unique id")
            obj = [bytes(uid.raw)]
            self.dist.broadcast_object_list(obj, src=0, group=self.group)
            h = ctypes.c_void_p()
            _lib.check(lib.tlb_ring_create(obj[0], self.Np, self.rank, int(device_index),
                                           ctypes.byref(h)), "ring create")
            self._ring = h
        return self._ring

    def close(self):
        if self._ring is not None:
            _lib.load().tlb_ring_destroy(self._ring)
            self._ring = None

    def abort_ring(self):
        """Release NCCL kernels stalled on a dead or late peer."""
        if self._ring is not None:
            _lib.load().tlb_ring_abort(self._ring)

    def async_error(self):
        """The ring communicator's asynchronous NCCL error code (0 = none)."""
        import ctypes
        if self._ring is None:
            return 0
        code = ctypes.c_int(0)
        _lib.check(_lib.load().tlb_ring_async_error(self._ring, ctypes.byref(code)),
                   "nccl async error")
        return code.value

    def start_face(self, w, step, axis, out_plus, out_minus):
        dist = self.dist
        nb = w.tile.neighbors
        if axis == "x":
            fwd, bwd = nb["right"], nb["left"]
            rin_p, rin_m = w.rbuf_plus, w.rbuf_minus
        else:
            fwd, bwd = nb["up"], nb["down"]
            rin_p, rin_m = w.rbuf_y_plus, w.rbuf_y_minus
        # same op order on every rank: each send is matched by the peer's
        # receive of the same direction, also when fwd == bwd
        ops = []
        if fwd is not None:
            ops.append(dist.P2POp(dist.isend, out_plus, fwd, self.group))
        if bwd is not None:
            ops.append(dist.P2POp(dist.irecv, rin_p, bwd, self.group))
        if bwd is not None:
            ops.append(dist.P2POp(dist.isend, out_minus, bwd, self.group))
        if fwd is not None:
            ops.append(dist.P2POp(dist.irecv, rin_m, fwd, self.group))
        return (dist.batch_isend_irecv(ops) if ops else []), (bwd is not None, fwd is not None)

    def finish_face(self, w, handle, axis, in_plus, in_minus, stream=None):
        # called under torch.cuda.stream(stream): wait() orders it after NCCL
        reqs, got = handle
        for req in reqs:
            try:
                req.wait()
            except Exception as exc:  # timeouts surface as DeadlockError
                raise DeadlockError(f"rank {w.tile.rank} stalled in the {axis.upper()} "
                                    f"exchange: {exc}", rank=w.tile.rank) from exc
        return list(got)

    def start_x(self, w, step, out_plus, out_minus):
        return self.start_face(w, step, "x", out_plus, out_minus)

    def finish_x(self, w, handle, in_plus, in_minus, stream=None):
        return self.finish_face(w, handle, "x", in_plus, in_minus, stream)

    def fail(self, rank, exc):
        self.failures.append((rank, exc))
        self.abort.set()


# ------------------------------------------------------------ rank worker --

@dataclass
class _StepRecord:
    step: int
    status: object      # device slice (bytes) of the per-step status ring
    events: tuple       # (t0, t1, t2, t3) CUDA events: comm / bulk / border,
                        # ("graph", e0, e1, G) for a replayed block, or None


class RankWorker:
    """One rank: owns a tile's double buffer in HBM and runs the step loop
    (runtime.py:163-404).

    ``fabric`` is a ``Fabric`` (in-process ranks) or ``DistFabric`` (one
    process per GPU).  ``device`` selects the GPU (default: current).  Both
    the 1-D X ring and the 2-D grid of ``decompose`` are supported; a step is
    three phases (``step_begin``/``step_mid``/``step_end``) so in-process
    ranks can be driven in lock step: Y faces are exchanged before X faces,
    whose full-height columns then carry the diagonal corners
    (runtime.py:8-12)."""

    _RING = 1024

    def __init__(self, tile, vs, params, fabric=None, schedule="staged", walls=True,
                 layout="column", halo=DEFAULT_HALO, debug_poison=False, device=None,
                 periodic_y=False, exchange="auto", timing="sampled", timing_every=32,
                 temporal="auto"):
        torch = _lib.torch_cuda()
        if schedule not in ("staged", "overlapped"):
            raise ConfigurationError(f"unknown schedule {schedule!r}")
        if exchange not in ("auto", "nccl", "p2p"):
            raise ConfigurationError(f"unknown exchange {exchange!r} (auto|nccl|p2p)")
        if timing not in ("sampled", "every", "off"):
            raise ConfigurationError(f"unknown timing {timing!r} (sampled|every|off)")
        if temporal not in ("auto", "on", "off"):
            raise ConfigurationError(f"unknown temporal {temporal!r} (auto|on|off)")
        self.temporal = temporal
        self.timing, self.timing_every, self._count = timing, max(1, int(timing_every)), 0
        self.tile = tile
        self.vs = vs
        self.params = params
        self.fabric = fabric
        self.schedule = schedule
        self.walls = walls
        self.periodic_y = periodic_y and not walls
        self.debug_poison = debug_poison
        self.device = torch.device(device) if device is not None else torch.device(
            "cuda", torch.cuda.current_device())
        # a 1-D ring rank that will pair steps across GPUs (tlb_peer_step2)
        # needs 6 X halo columns: both steps' pull reach
        order0 = params.eq_order if params.eq_order is not None else vs.eq_order
        nb0 = tile.neighbors
        ring_1d = (nb0["left"] != tile.rank and tile.grid[1] == 1)
        self.pair_ring_wanted = (
            ring_1d and schedule == "overlapped" and exchange in ("auto", "p2p")
            and vs.Q == 37 and order0 == 4 and tile.Lx >= 12 and tile.Ly >= 8
            and not debug_poison and temporal != "off"
            and (temporal == "on" or (params.arith == "fast"
                                      and tile.Lx * tile.Ly >= self.PAIR_MIN_SITES)))
        hx = max(halo, 6) if self.pair_ring_wanted else halo
        self.geom = LatticeGeometry(tile.Lx, tile.Ly, hx, halo, vs.Q, layout)
        self.halo = halo
        nb = tile.neighbors
        self.x_self = nb["left"] == tile.rank
        # Y: ring onto itself (one row of ranks, periodic), or exchange with
        # up/down neighbours (2-D), or walls
        self.y_self = tile.grid[1] == 1 and nb["up"] is not None
        self.ex_up = nb["up"] is not None and not self.y_self
        self.ex_down = nb["down"] is not None and not self.y_self
        self.y_exchange = self.ex_up or self.ex_down
        self.wall_bot = walls and tile.lowermost
        self.wall_top = walls and tile.uppermost
        with torch.cuda.device(self.device):
            _lib.ensure_stencil(vs, self.device.index)
            self.prv, self.nxt = allocate_field(self.geom, vs, device=self.device)
            self.stream = torch.cuda.Stream(self.device)
            self.comm_stream = torch.cuda.Stream(self.device, priority=-1)
            lib = _lib.load()
            n = int(lib.tlb_face_payload_len(field_desc(self.prv)))
            ny_ = int(lib.tlb_face_payload_len_y(field_desc(self.prv)))
            self.payload_len, self.payload_len_y = n, ny_
            self.rbuf_plus = torch.empty(n, dtype=torch.float64, device=self.device)
            self.rbuf_minus = torch.empty(n, dtype=torch.float64, device=self.device)
            self.rbuf_y_plus = torch.empty(ny_, dtype=torch.float64, device=self.device)
            self.rbuf_y_minus = torch.empty(ny_, dtype=torch.float64, device=self.device)
            self._ring = None
            if isinstance(fabric, DistFabric) and fabric.native and fabric.Np > 1:
                import ctypes
                self._ring = fabric.ring(self.device.index)
                # two X payloads (+ a step tag each), four Y payloads (ditto)
                self.sbuf2 = torch.empty(2 * (n + 1), dtype=torch.float64, device=self.device)
                self.rbuf2 = torch.empty(2 * (n + 1), dtype=torch.float64, device=self.device)
                self.ybuf4 = torch.empty(4 * (ny_ + 1), dtype=torch.float64, device=self.device)
                _lib.check(lib.tlb_ring_set_neighbors(
                    self._ring, nb["left"], nb["right"],
                    nb["up"] if self.ex_up else -1, nb["down"] if self.ex_down else -1,
                    ctypes.c_void_p(self.ybuf4.data_ptr())), "ring neighbours")
            self._status_ring = torch.zeros((self._RING, _lib.STATUS_BYTES),
                                            dtype=torch.uint8, device=self.device)
            self._graphs = {}
            self._gstatus = None
            self._capture_slot = None
            self._peer = None
            # NVLink peer stores fused into the step kernel (tlb_peer_step):
            # 1-D ring or 2-D grid, overlapped schedule, the specialised
            # D2Q37 order-4 kernels, tiles at least 7 sites across every
            # exchanged direction.  "auto" takes it when it applies, else
            # the NCCL ring; "p2p" insists.
            order = params.eq_order if params.eq_order is not None else vs.eq_order
            # in-process ranks (Fabric) link their peers once all tiles exist
            # (link_local_peers); one process per GPU maps them over CUDA IPC
            self.peer_capable = ((not self.x_self or self.y_exchange)
                                 and schedule == "overlapped" and vs.Q == 37 and order == 4
                                 and (self.x_self or tile.Lx >= 7)
                                 and (not self.y_exchange or tile.Ly >= 7))
            peer_ok = self._ring is not None and self.peer_capable
            self.exchange = exchange
            if exchange == "p2p" and not peer_ok and self._ring is not None:
                raise ConfigurationError(
                    "exchange='p2p' needs D2Q37 order-4 tiles >= 7 sites across each "
                    "exchanged direction with the overlapped schedule")
            if exchange in ("auto", "p2p") and peer_ok:
                self._setup_peer(fabric, strict=exchange == "p2p")
            # order the allocations' zero-fills before any work on our stream
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
        self.plans = face_plans(vs, halo)
        self.tparams = _lib.params(params, vs)
        self.exchange_mode = ("p2p" if self._peer is not None else
                              "nccl" if self._ring is not None else
                              "self" if self.x_self and not self.y_exchange else "fabric")
        self._records = []
        self._retained = []
        self._metrics = []
        self.snapshots = []
        self._halo_depth = 0    # peer halos filled: 0 no, 3 single-step, 6 pair depth

    def _setup_peer(self, fabric, strict=False):
        """Map the ring neighbours' field buffers and mailboxes (CUDA IPC over
        NVLink) for the fused peer-memory step (csrc/tlb_peer.cuh).

        Collective: if any rank cannot export or open the IPC mappings, every
        rank falls back to the NCCL ring together (or, with strict=True,
        i.e. exchange="p2p", every rank raises DeviceError)."""
        import ctypes
        import warnings
        torch = _lib.torch_cuda()
        lib = _lib.load()
        # [0..7] step published by the neighbour in direction d (written by
        # them), [8] this rank's border-block counter, [9] sticky timeout
        # flag (csrc/tlb_peer.cuh)
        self.mailbox = torch.zeros(16, dtype=torch.int64, device=self.device)
        torch.cuda.synchronize(self.device)

        def agree(ok, why):
            votes = [None] * fabric.Np
            fabric.dist.all_gather_object(votes, (ok, why), group=fabric.group)
            bad = [f"rank {r}: {w}" for r, (o, w) in enumerate(votes) if not o]
            if bad and strict:
                raise DeviceError("peer-store exchange unavailable: " + "; ".join(bad))
            if bad:
                warnings.warn("peer-store exchange unavailable, using the NCCL ring: "
                              + "; ".join(bad))
            return not bad

        mine, why = [], ""
        try:
            for t in (self.prv.data, self.nxt.data, self.mailbox):
                h = ctypes.create_string_buffer(64)
                off = ctypes.c_int64(0)
                _lib.check(lib.tlb_ipc_handle(t.data_ptr(), h, ctypes.byref(off)),
                           "ipc handle")
                mine.append((bytes(h.raw), int(off.value)))
        except ThermoLBError as exc:
            mine, why = None, str(exc)
        allinfo = [None] * fabric.Np
        fabric.dist.all_gather_object(allinfo, mine, group=fabric.group)
        if not agree(mine is not None, why):
            return
        ranks = self._peer_neighbours()
        blank = (b"\0" * 64, 0)
        order = [item for r in ranks for item in (allinfo[r] if r is not None else [blank] * 3)]
        handles = b"".join(h for h, _ in order)
        offs = (ctypes.c_int64 * 24)(*[o for _, o in order])
        present = (ctypes.c_int * 8)(*[int(r is not None) for r in ranks])
        hp = ctypes.c_void_p()
        try:
            _lib.check(lib.tlb_peer_create2(self.device.index, handles, offs, present,
                                            ctypes.byref(hp)), "peer create")
            ok, why = True, ""
        except ThermoLBError as exc:
            ok, why = False, str(exc)
        if not agree(ok, why):
            if ok:
                lib.tlb_peer_destroy(hp)
            return
        self._adopt_peer(hp, getattr(fabric, "timeout", None))
        fabric.dist.barrier(group=fabric.group)

    def _adopt_peer(self, hp, timeout):
        """Start stepping through the peer object hp (buffer A = prv now)."""
        torch = _lib.torch_cuda()
        if timeout:
            _lib.check(_lib.load().tlb_peer_set_timeout(hp, float(timeout)), "peer timeout")
        self._peer = hp
        self._bufA = self.prv.data.data_ptr()
        self._peer_step = 0
        self._last_tag = None
        self._halo_depth = 0
        if self.debug_poison:
            # both buffers' halos start poisoned; afterwards every peer step
            # re-poisons prv's halos once its border blocks have read them
            # (TLB_F_POISON_HALOS), before any neighbour may store into them
            self._poison_halos(self.prv)
            self._poison_halos(self.nxt)
        torch.cuda.synchronize(self.device)

    # the eight directions of csrc/tlb_peer.cuh: (dx, dy)
    _PEER_DIRS = ((-1, 0), (1, 0), (0, -1), (0, 1), (-1, -1), (1, -1), (-1, 1), (1, 1))

    def _peer_neighbours(self):
        """Rank of the neighbour in each peer direction, None where that side
        is not exchanged (self-periodic X or Y, or a wall)."""
        nx, ny = self.tile.grid
        ix, iy = self.tile.coords
        out = []
        for dx, dy in self._PEER_DIRS:
            if (dx and self.x_self) or (dy < 0 and not self.ex_down) or \
                    (dy > 0 and not self.ex_up):
                out.append(None)
                continue
            out.append(((iy + dy) % ny) * nx + (ix + dx) % nx)
        return out

    # -- helpers -------------------------------------------------------------
    @property
    def Np(self):
        return self.tile.grid[0] * self.tile.grid[1]

    @property
    def self_ring(self):
        return self.x_self

    def _sp(self, stream=None):
        return (stream or self.stream).cuda_stream

    def _check(self, code, what):
        _lib.check(code, what)

    def _flags(self):
        """Fused-kernel flags of this rank (walls, implicit halos, monitor)."""
        f = _lib.F_COUNT_NEG
        if self.wall_bot:
            f |= _lib.F_WALL_BOT | _lib.F_CLAMP_BOT
        if self.wall_top:
            f |= _lib.F_WALL_TOP | _lib.F_CLAMP_TOP
        if self.y_self:
            f |= _lib.F_WRAP_Y
        if self.x_self:
            f |= _lib.F_WRAP_X
        return f

    def _ymode(self):
        """How pack_x sources the Y halo rows (tlb_pack_x)."""
        if self.wall_bot and self.wall_top:
            return 1
        if self.y_self:
            return 2
        if self.wall_bot:
            return 3
        if self.wall_top:
            return 4
        return 0

    def _rec(self, ev, k):
        if ev is not None:
            ev[k].record(self.stream)

    def _status_slot(self):
        if self._capture_slot is not None:
            return self._capture_slot
        if len(self._records) >= self._RING:
            self.collect()
        return self._status_ring[len(self._records)]

    def retain(self, t):
        self._retained.append(t)

    # -- halo exchange (reference names) -------------------------------------
    def pack_x(self, f, sign, ymode=0, stream=None):
        """Outgoing X-face payload (runtime.py:199-208); a new device tensor."""
        torch = _lib.torch_cuda()
        with torch.cuda.stream(stream or self.stream):
            buf = torch.empty(self.payload_len, dtype=torch.float64, device=self.device)
        self._check(_lib.load().tlb_pack_x(field_desc(f), int(sign), int(ymode),
                                           buf.data_ptr(), self._sp(stream)), "pack_x")
        return buf

    def unpack_x(self, f, sign, payload, stream=None):
        """Scatter a received X payload into the halo columns (runtime.py:210-224)."""
        torch = _lib.torch_cuda()
        if not isinstance(payload, torch.Tensor):
            payload = torch.as_tensor(np.asarray(payload, dtype=np.float64), device=self.device)
        if payload.numel() != self.payload_len:
            raise ProtocolError(f"rank {self.tile.rank}: X payload size mismatch")
        self._check(_lib.load().tlb_unpack_x(field_desc(f), int(sign), payload.data_ptr(),
                                             self._sp(stream)), "unpack_x")

    def pack_y(self, f, sign, stream=None):
        """Outgoing Y-face payload, physical columns only (runtime.py:226-235)."""
        torch = _lib.torch_cuda()
        with torch.cuda.stream(stream or self.stream):
            buf = torch.empty(self.payload_len_y, dtype=torch.float64, device=self.device)
        self._check(_lib.load().tlb_pack_y(field_desc(f), int(sign), buf.data_ptr(),
                                           self._sp(stream)), "pack_y")
        return buf

    def unpack_y(self, f, sign, payload, stream=None):
        """Scatter a received Y payload into the halo rows (runtime.py:237-246)."""
        torch = _lib.torch_cuda()
        if not isinstance(payload, torch.Tensor):
            payload = torch.as_tensor(np.asarray(payload, dtype=np.float64), device=self.device)
        if payload.numel() != self.payload_len_y:
            raise ProtocolError(f"rank {self.tile.rank}: Y payload size mismatch")
        self._check(_lib.load().tlb_unpack_y(field_desc(f), int(sign), payload.data_ptr(),
                                             self._sp(stream)), "unpack_y")

    def _start(self, axis, step, f, ymode=0, stream=None):
        torch = _lib.torch_cuda()
        stream = stream or self.stream
        if axis == "x":
            out = (self.pack_x(f, 1, ymode, stream), self.pack_x(f, -1, ymode, stream))
        else:
            out = (self.pack_y(f, 1, stream), self.pack_y(f, -1, stream))
        with torch.cuda.stream(stream):
            return self.fabric.start_face(self, step, axis, *out)

    def _finish(self, axis, f, handle, stream=None):
        torch = _lib.torch_cuda()
        stream = stream or self.stream
        bufs = ((self.rbuf_plus, self.rbuf_minus) if axis == "x"
                else (self.rbuf_y_plus, self.rbuf_y_minus))
        with torch.cuda.stream(stream):
            got = self.fabric.finish_face(self, handle, axis, *bufs, stream)
        unpack = self.unpack_x if axis == "x" else self.unpack_y
        if got[0]:
            unpack(f, 1, bufs[0], stream)
        if got[1]:
            unpack(f, -1, bufs[1], stream)

    def pbc_nc(self, f, step):
        """Exchange the Y halo rows (runtime.py:264-267)."""
        if self.y_self:
            self._check(_lib.load().tlb_pbc_self_y(field_desc(f), self._sp()), "pbc_nc")
        elif self.y_exchange:
            self._finish("y", f, self._start("y", step, f))

    def pbc_c(self, f, step):
        """Exchange the X halo columns around the ring (runtime.py:281-284)."""
        if self.x_self:
            self._check(_lib.load().tlb_pbc_self_x(field_desc(f), self._sp()), "pbc_c")
            return
        self._finish("x", f, self._start("x", step, f))

    def _extend_wall_halos(self, f):
        """runtime.py:296-305."""
        if self.wall_top or self.wall_bot:
            self._check(_lib.load().tlb_extend_walls(field_desc(f), int(self.wall_top),
                                                     int(self.wall_bot), self._sp()),
                        "extend_walls")

    def _poison_halos(self, f):
        """runtime.py:288-294 (debug mode only)."""
        torch = _lib.torch_cuda()
        g = self.geom
        p = f.pops
        with torch.cuda.stream(self.stream):
            p[:, :g.Hx, :] = float("nan")
            p[:, g.Hx + g.Lx:, :] = float("nan")
            p[:, :, :g.Hy] = float("nan")
            p[:, :, g.Hy + g.Ly:] = float("nan")

    def _bc_rows(self):
        g = self.geom
        rows = []
        if self.wall_bot:
            rows.append((g.Hy, g.Hy + WALL_ROWS))
        if self.wall_top:
            rows.append((g.Hy + g.Ly - WALL_ROWS, g.Hy + g.Ly))
        return rows

    # -- schedules -----------------------------------------------------------
    def _fused(self, x0, x1, y0, y1, flags, st, stream=None):
        if x1 <= x0 or y1 <= y0:
            return
        self._check(_lib.load().tlb_fused(
            field_desc(self.prv), field_desc(self.nxt), _lib.region(x0, x1, y0, y1),
            self.tparams, flags, st, self._sp(stream)), "fused")

    def _bulk_rect(self):
        """Sites that need no exchanged halo (RankWorker._frame_slices,
        runtime.py:326-338): 3 away from exchanged X and Y edges."""
        g, h = self.geom, self.halo
        x0, x1 = g.Hx, g.Hx + g.Lx
        if not self.x_self:
            x0, x1 = g.Hx + h, max(g.Hx + h, g.Hx + g.Lx - h)
        y0 = min(g.Hy + (h if self.ex_down else 0), g.Hy + g.Ly)
        y1 = max(y0, g.Hy + g.Ly - (h if self.ex_up else 0))
        return x0, x1, y0, y1

    def _frames(self, flags, st, stream):
        """The bands around the bulk rectangle, after the exchanges."""
        g = self.geom
        X0, X1, Y0, Y1 = g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly
        x0, x1, y0, y1 = self._bulk_rect()
        if x1 <= x0:   # tile narrower than two borders: everything is frame
            self._fused(X0, X1, Y0, Y1, flags, st, stream)
            return
        self._fused(X0, x0, Y0, Y1, flags, st, stream)
        self._fused(x1, X1, Y0, Y1, flags, st, stream)
        self._fused(x0, x1, Y0, y0, flags, st, stream)
        self._fused(x0, x1, y1, Y1, flags, st, stream)

    def step(self, step_no):
        """One time step (runtime.py:355-400), enqueued on the rank's streams."""
        self.step_begin(step_no)
        self.step_mid(step_no)
        self.step_end(step_no)

    # -- CUDA-graph replay of the step sequence ------------------------------
    GRAPH_STEPS = 32    # even: the buffer roles return to the captured ones

    def graphable(self):
        """A single self-periodic tile (no exchange with other ranks): its
        whole step is a fixed launch sequence on self.stream."""
        return (self.x_self and not self.y_exchange and self._ring is None
                and self._peer is None and not self.debug_poison and self.timing != "every")

    # "auto" pairs steps only on tiles this large: the two-step kernel needs
    # enough strip runs to fill the GPU (512x1024: 10.3k vs 9.8k MLUPS for
    # the single step, 1024x1024: 11.0k vs 10.2k, 1024x2048: 12.7k vs 10.6k;
    # 512x256 and 256x128 lose; profiles/r02_tb2.md)
    PAIR_MIN_SITES = 500_000

    def pairable(self):
        """Two steps per launch (temporal blocking, csrc/tb2.cu): a single
        self-periodic tile with the overlapped schedule, D2Q37 order 4, at
        least 8x8.  "auto" takes it for the fast arithmetic on large tiles
        (where it is the faster kernel); "on" for both arithmetics and any
        size; results are the same bits as two single steps either way."""
        if self.temporal == "off" or self.schedule != "overlapped" or self.debug_poison:
            return False
        order = self.params.eq_order if self.params.eq_order is not None else self.vs.eq_order
        if self._peer is not None:
            # across GPUs on the 1-D ring (tlb_peer_step2): decided with the
            # halo width at construction
            return (self.pair_ring_wanted and self.geom.Hx >= 6 and not self.y_exchange
                    and (self.temporal == "on" or self.tparams.arith == _lib.ARITH["fast"]))
        if not (self.x_self and not self.y_exchange and self._ring is None and self._peer is None
                and (self.y_self or (self.wall_bot and self.wall_top))
                and self.vs.Q == 37 and order == 4 and self.geom.Lx >= 8 and self.geom.Ly >= 8):
            return False
        return self.temporal == "on" or (self.tparams.arith == _lib.ARITH["fast"] and
                                         self.geom.Lx * self.geom.Ly >= self.PAIR_MIN_SITES)

    def prime_halos(self, step_no, depth, status=None):
        """Peer-store exchange: make prv's X halos `depth` deep (3: the face
        plans, for single steps; 6: for step pairs) before step step_no --
        the border sites push their values into the neighbours' halos as if
        step_no-1 had just run (counts as a peer step).  A no-op when the
        halos already are that deep; step()/step_pair() call it themselves,
        in-process lock-step drivers call it for every rank first so that
        no rank's first step waits on a prime launched after it."""
        if self._peer is None or self._halo_depth >= depth:
            return
        lib = _lib.load()
        if status is None:
            status = self._status_slot().data_ptr()
        prv_index = 0 if self.prv.data.data_ptr() == self._bufA else 1
        fn = lib.tlb_peer_prime2 if depth > 3 else lib.tlb_peer_prime
        self._check(fn(self._peer, field_desc(self.prv), prv_index, self.tparams, status,
                       self.mailbox.data_ptr(), self._peer_step, step_no - 1, self._sp()),
                    "peer prime")
        self._peer_step += 1
        self._last_tag = step_no - 1
        self._halo_depth = max(depth, 3)

    def step_pair(self, step_no):
        """Steps step_no and step_no + 1 in ONE launch (tlb_step2_self): the
        intermediate state stays in shared memory.  Bitwise equal to
        step(step_no); step(step_no + 1); per-step metrics and failures keep
        their step numbers."""
        torch = _lib.torch_cuda()
        if self._capture_slot is not None:
            s1, s2 = self._capture_slot
        else:
            if len(self._records) + 2 > self._RING:
                self.collect()
            n = len(self._records)
            s1, s2 = self._status_ring[n], self._status_ring[n + 1]
        timed = self.timing == "every" or (
            self.timing == "sampled" and self._count % self.timing_every == 0)
        self._count += 2
        ev = None
        if timed:
            ev = ("graph", torch.cuda.Event(enable_timing=True),
                  torch.cuda.Event(enable_timing=True), 2)
            ev[1].record(self.stream)
        lib = _lib.load()
        if self._peer is not None:
            self.prime_halos(step_no, 6, s1.data_ptr())
            nxt_index = 0 if self.nxt.data.data_ptr() == self._bufA else 1
            self._check(lib.tlb_peer_step2(
                self._peer, field_desc(self.prv), field_desc(self.nxt), nxt_index,
                self.tparams, self._flags(), s1.data_ptr(), s2.data_ptr(),
                self.mailbox.data_ptr(), self._peer_step, step_no,
                int(self._last_tag == step_no - 1), self._sp()), "peer step2")
            self._peer_step += 1
            self._last_tag = step_no + 1
            self._halo_depth = 6
        else:
            self._check(lib.tlb_step2_self(
                field_desc(self.prv), field_desc(self.nxt), self.tparams, int(self.wall_bot),
                int(self.y_self), 1, s1.data_ptr(), s2.data_ptr(), int(step_no), self._sp()),
                "step2")
        if ev is not None:
            ev[2].record(self.stream)
        self._records.append(_StepRecord(step_no, s1, ev))
        self._records.append(_StepRecord(step_no + 1, s2, ev))
        self.prv, self.nxt = swap_buffers(self.prv, self.nxt)

    def run_steps(self, step0, n):
        """Steps step0 .. step0+n-1, bitwise identical to calling step().

        On a graphable tile the launch sequence of GRAPH_STEPS steps is
        captured once per buffer parity into a CUDA graph and replayed: the
        per-step host cost (~60 us of Python + ctypes) otherwise dominates
        small lattices (C1 256x128: ~5 us of GPU work per step).  Each
        replay writes its per-step status blocks to a staging array that is
        copied into the status ring, so metrics and per-site errors (with
        their step numbers) surface at collect() exactly as with step()."""
        G = self.GRAPH_STEPS
        s, end = step0, step0 + n
        if self.graphable() and n >= G:
            torch = _lib.torch_cuda()
            while end - s >= G:
                graph = self._graph_for()
                if len(self._records) + G > self._RING:
                    self.collect()
                pos = len(self._records)
                ev = None
                if self.timing != "off":
                    # one event pair per replay: every step of the block
                    # reports the block's average step time as t_bulk
                    ev = ("graph", torch.cuda.Event(enable_timing=True),
                          torch.cuda.Event(enable_timing=True), G)
                    ev[1].record(self.stream)
                with torch.cuda.stream(self.stream):
                    graph.replay()
                    self._status_ring[pos:pos + G].copy_(self._gstatus)
                if ev is not None:
                    ev[2].record(self.stream)
                self._records.extend(_StepRecord(s + j, self._status_ring[pos + j], ev)
                                     for j in range(G))
                s += G
        pair = self.pairable()
        while s < end:
            if pair and end - s >= 2:
                self.step_pair(s)
                s += 2
            else:
                self.step(s)
                s += 1

    def _graph_for(self):
        key = (self.prv.data.data_ptr(), self._flags(), self.schedule, self.pairable(),
               bytes(self.tparams))
        graph = self._graphs.get(key)
        if graph is None:
            graph = self._graphs[key] = self._capture()
        return graph

    def _capture(self):
        torch = _lib.torch_cuda()
        G = self.GRAPH_STEPS
        if self._gstatus is None:
            self._gstatus = torch.zeros((G, _lib.STATUS_BYTES), dtype=torch.uint8,
                                        device=self.device)
        saved = (self._records, self._count, self.timing)
        self._records, self.timing = [], "off"
        graph = torch.cuda.CUDAGraph()
        # capture_begin/end directly: the torch.cuda.graph context manager
        # also runs gc.collect() and empty_cache(), which cost tens of ms and
        # force later allocations back to cudaMalloc
        try:
            with torch.cuda.stream(self.stream):
                graph.capture_begin(capture_error_mode="thread_local")
                try:
                    self._gstatus.zero_()
                    pair = self.pairable()
                    j = 0
                    while j < G:
                        if pair:
                            self._capture_slot = (self._gstatus[j], self._gstatus[j + 1])
                            self.step_pair(j)
                            j += 2
                        else:
                            self._capture_slot = self._gstatus[j]
                            self.step(j)
                            j += 1
                finally:
                    graph.capture_end()
        finally:
            self._capture_slot = None
            self._records, self._count, self.timing = saved
        return graph

    def step_begin(self, step_no):
        torch = _lib.torch_cuda()
        g = self.geom
        lib = _lib.load()
        slot = self._status_slot()
        st = slot.data_ptr()
        # per-step timing events cost ~10 us of GPU time per step (measured,
        # tools/gap_probe.py): by default only every `timing_every`-th step
        # is timed; the others report NaN times (negatives are always exact)
        timed = self.timing == "every" or (
            self.timing == "sampled" and self._count % self.timing_every == 0)
        self._count += 1
        ev = tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) if timed else None
        self._pending = (step_no, slot, ev, st)
        self._hy = self._hx = None
        self._bulk_timed = False
        self._rec(ev, 0)
        if self.debug_poison and self._peer is None:
            self._poison_halos(self.prv)
        if self.schedule == "staged":
            # the reference's order: wall extension, Y halos, X halos
            self._extend_wall_halos(self.prv)
            if self._ring is not None:
                self._check(lib.tlb_ring_exchange(
                    self._ring, field_desc(self.prv), 0, self.sbuf2.data_ptr(),
                    self.rbuf2.data_ptr(), self._sp()), "ring exchange")
            elif self.y_self:
                self._check(lib.tlb_pbc_self_y(field_desc(self.prv), self._sp()), "pbc_nc")
            elif self.y_exchange:
                self._hy = self._start("y", step_no, self.prv)
            return
        flags = self._flags()
        self._flags_now = flags
        if self._peer is not None:
            self.prime_halos(step_no, 3, st)
            nxt_index = 0 if self.nxt.data.data_ptr() == self._bufA else 1
            pflags = flags | (_lib.F_POISON_HALOS if self.debug_poison else 0)
            self._rec(ev, 1)
            self._check(lib.tlb_peer_step(
                self._peer, field_desc(self.prv), field_desc(self.nxt), nxt_index,
                self.tparams, pflags, st, self.mailbox.data_ptr(), self._peer_step,
                step_no, int(self._last_tag == step_no - 1), self._sp()), "peer step")
            self._peer_step += 1
            self._last_tag = step_no
            self._halo_depth = 3      # a single step refills only the face-plan lines
            self._rec(ev, 2)
            self._bulk_timed = True
            return
        if self._ring is not None:
            self._rec(ev, 1)
            self._rec(ev, 2)
            self._check(lib.tlb_ring_step(
                self._ring, field_desc(self.prv), field_desc(self.nxt), self.tparams,
                flags & ~_lib.F_WRAP_X, st, self.sbuf2.data_ptr(), self.rbuf2.data_ptr(),
                ev[1].cuda_event if ev else None, ev[2].cuda_event if ev else None,
                step_no, self._sp()), "ring step")
            self._bulk_timed = True
            return
        if self.x_self and not self.y_exchange:
            # one fused launch is the whole step (implicit periodic X halo)
            self._rec(ev, 1)
            self._fused(g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly, flags, st)
            self._rec(ev, 2)
            self._bulk_timed = True
            return
        # faces out on the high-priority side stream (after prv is complete),
        # bulk on the main stream concurrently
        cs = self.comm_stream
        cs.wait_stream(self.stream)
        if self.y_exchange:
            self._hy = self._start("y", step_no, self.prv, stream=cs)
        elif not self.x_self:
            self._hx = self._start("x", step_no, self.prv, self._ymode(), stream=cs)
        self._rec(ev, 1)
        self._fused(*self._bulk_rect(), flags, st)
        self._rec(ev, 2)
        self._bulk_timed = True

    def step_mid(self, step_no):
        """Y halos in, then X faces out (2-D); nothing to do on a 1-D ring."""
        if self._hy is None:
            if self.schedule == "staged" and self._ring is None and self._hx is None:
                if self.x_self:
                    self._check(_lib.load().tlb_pbc_self_x(field_desc(self.prv), self._sp()),
                                "pbc_c")
                else:
                    self._hx = self._start("x", step_no, self.prv)
            return
        stream = self.comm_stream if self.schedule == "overlapped" else self.stream
        self._finish("y", self.prv, self._hy, stream)
        self._hy = None
        if self.x_self:
            if self.schedule == "staged":
                self._check(_lib.load().tlb_pbc_self_x(field_desc(self.prv), self._sp()),
                            "pbc_c")
            return
        ymode = 0 if self.schedule == "staged" else self._ymode()
        self._hx = self._start("x", step_no, self.prv, ymode, stream=stream)

    def step_end(self, step_no):
        g = self.geom
        lib = _lib.load()
        step_no_, slot, ev, st = self._pending
        if self.schedule == "staged":
            if self._hx is not None:
                self._finish("x", self.prv, self._hx)
                self._hx = None
            self._rec(ev, 1)
            self._rec(ev, 2)
            full = _lib.region(g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly)
            self._check(lib.tlb_propagate(field_desc(self.prv), field_desc(self.nxt), full,
                                          self._sp()), "propagate")
            if self.wall_top or self.wall_bot:
                self._check(lib.tlb_bc(field_desc(self.nxt), self.tparams, int(self.wall_top),
                                       int(self.wall_bot), g.Hx, g.Hx + g.Lx, st, self._sp()),
                            "bc")
            self._check(lib.tlb_collide(field_desc(self.nxt), field_desc(self.nxt), full,
                                        self.tparams, _lib.F_COUNT_NEG, st, self._sp()),
                        "collide")
        elif (self._ring is None and self._peer is None
              and not (self.x_self and not self.y_exchange)):
            # halos in -> frame bands on the side stream, concurrent with bulk
            cs = self.comm_stream
            if self._hx is not None:
                self._finish("x", self.prv, self._hx, cs)
                self._hx = None
            self._frames(self._flags_now, st, cs)
            self.stream.wait_stream(cs)
        self._rec(ev, 3)
        self._records.append(_StepRecord(step_no, slot, ev))
        self.prv, self.nxt = swap_buffers(self.prv, self.nxt)

    # -- results -------------------------------------------------------------
    def synchronize(self, timeout=None):
        """Wait for this rank's queued steps.  With a fabric timeout (one
        process per GPU) a rank that waits longer than `timeout` seconds --
        a stalled or failed ring neighbour -- aborts the NCCL ring and raises
        DeadlockError naming itself (runtime.py:146-149)."""
        torch = _lib.torch_cuda()
        if timeout is None:
            timeout = getattr(self.fabric, "timeout", None) if isinstance(
                self.fabric, DistFabric) else None
        if not timeout:
            self.stream.synchronize()
            return
        if self._peer is not None:
            # the step kernel's own bounded wait (the same timeout) reports
            # a stalled neighbour first, with its step; then later queued
            # steps fail at once
            timeout = 1.5 * timeout + 1.0
        ev = torch.cuda.Event()
        ev.record(self.stream)
        deadline = time.monotonic() + timeout
        while not ev.query():
            if time.monotonic() > deadline:
                err = self.fabric.async_error()
                self.fabric.abort_ring()
                raise DeadlockError(f"rank {self.tile.rank} stalled for {timeout:.0f} s waiting "
                                    f"for its ring neighbours (NCCL async error {err})",
                                    rank=self.tile.rank)
            time.sleep(2e-4)

    def close(self):
        """Release the peer mappings (after every rank finished its steps)."""
        if getattr(self, "_peer", None) is not None:
            self.synchronize()
            _lib.load().tlb_peer_destroy(self._peer)
            self._peer = None

    def collect(self, raise_errors=True):
        """Materialise pending per-step metrics (one host sync) and raise the
        first per-site failure the kernels flagged, like the reference's
        in-step exceptions (kernels.py:62-66, 134-135, 85-86)."""
        if not self._records:
            return
        self.synchronize()
        n = len(self._records)
        raw = self._status_ring[:n].cpu().numpy()
        # the status blocks as one structured array (flags, negatives):
        # per-step ctypes copies cost more than the small-tile steps
        flags = raw[:, _lib.STATUS_FLAGS_OFF:_lib.STATUS_FLAGS_OFF + 4].copy().view(np.uint32)[:, 0]
        negs = raw[:, _lib.STATUS_NEG_OFF:_lib.STATUS_NEG_OFF + 8].copy().view(np.uint64)[:, 0]
        bad = np.flatnonzero(flags)
        err = None
        if len(bad):
            i = int(bad[0])
            err = (self._records[i].step, _lib.TlbStatus.from_buffer_copy(raw[i].tobytes()))
        span = {}          # one elapsed_time per launch (block), not per step
        nan = float("nan")
        for rec, neg in zip(self._records, negs.tolist()):
            if rec.events is None:
                self._metrics.append({"t_comm_nc": nan, "t_comm_c": nan, "t_bulk": nan,
                                      "t_border": nan, "negatives": neg})
                continue
            if rec.events[0] == "graph":
                key = id(rec.events)
                t = span.get(key)
                if t is None:
                    _, g0, g1, nsteps = rec.events
                    t = span[key] = g0.elapsed_time(g1) * 1e-3 / nsteps
                self._metrics.append({"t_comm_nc": 0.0, "t_comm_c": 0.0, "t_bulk": t,
                                      "t_border": 0.0, "negatives": neg})
                continue
            t0, t1, t2, t3 = rec.events
            if self.schedule == "staged":
                m = {"t_comm_nc": 0.0, "t_comm_c": t0.elapsed_time(t1) * 1e-3,
                     "t_bulk": t2.elapsed_time(t3) * 1e-3, "t_border": 0.0}
            else:
                m = {"t_comm_nc": 0.0, "t_comm_c": t0.elapsed_time(t1) * 1e-3,
                     "t_bulk": t1.elapsed_time(t2) * 1e-3,
                     "t_border": t2.elapsed_time(t3) * 1e-3}
            m["negatives"] = neg
            self._metrics.append(m)
        self._records = []
        self._retained = []
        with _lib.torch_cuda().cuda.stream(self.stream):
            self._status_ring.zero_()
        if err is not None and raise_errors:
            step, s = err
            if s.flags & _lib.ST_PROTOCOL:
                raise ProtocolError(f"rank {self.tile.rank} step {step}: a neighbour's halo "
                                    "carries another step's tag")
            if s.flags & _lib.ST_PEER_TIMEOUT:
                raise DeadlockError(f"rank {self.tile.rank} step {step}: a ring neighbour did "
                                    "not publish its step (peer-memory exchange)",
                                    rank=self.tile.rank)
            if s.flags & _lib.ST_EQ_DOMAIN:
                raise DomainError(f"rank {self.tile.rank} step {step}: "
                                  "equilibrium requires rho > 0 and T > 0")
            if s.flags & _lib.ST_DEGENERATE:
                site = [int(s.site_x[0]), int(s.site_y[0])]
                raise DegenerateStateError(
                    f"rank {self.tile.rank} step {step}: non-positive density at [{site}]",
                    sites=np.array([site]))
            raise DomainError(f"rank {self.tile.rank} step {step}: shifted temperature "
                              "T_bar <= 0")

    @property
    def metrics(self):
        self.collect()
        return self._metrics

    def physical_block(self):
        """(Q, Lx, Ly) device copy of the current state (runtime.py:402-404),
        ordered before later work on the caller's current stream."""
        torch = _lib.torch_cuda()
        g = self.geom
        with torch.cuda.stream(self.stream):
            out = self.prv.pops[:, g.phys_x, g.phys_y].contiguous()
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return out

    def load_block(self, block):
        """prv[phys] = block (sim.py:74-75); block is (Q, Lx, Ly)."""
        torch = _lib.torch_cuda()
        self._halo_depth = 0
        g = self.geom
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            src = block if isinstance(block, torch.Tensor) else torch.as_tensor(
                np.ascontiguousarray(block, dtype=np.float64))
            self.prv.pops[:, g.phys_x, g.phys_y].copy_(src, non_blocking=True)
            if src.is_cuda and src.device == self.device:
                src.record_stream(self.stream)


def link_local_peers(workers, strict=False):
    """Peer stores for in-process ranks (the Fabric's simulated ranks,
    runtime.py:116-160): every tile's step kernel stores its border
    populations straight into its neighbours' halos and publishes the step
    through a device mailbox (csrc/tlb_peer.cuh) -- the kernel of one process
    per GPU, with plain device pointers instead of CUDA IPC.  `workers` must
    hold every rank.  Returns True when linked; with strict=False the ranks
    keep the Fabric exchange when the peer step does not apply."""
    import ctypes
    torch = _lib.torch_cuda()
    by_rank = {w.tile.rank: w for w in workers}
    ok = (len(workers) > 1 and all(w.peer_capable for w in workers)
          and len(by_rank) == workers[0].Np and all(w._peer is None for w in workers))
    if not ok:
        if strict:
            raise ConfigurationError(
                "exchange='p2p' needs D2Q37 order-4 tiles >= 7 sites across each exchanged "
                "direction with the overlapped schedule, and every rank in this process")
        return False
    lib = _lib.load()
    for w in workers:
        with torch.cuda.device(w.device):
            w.mailbox = torch.zeros(16, dtype=torch.int64, device=w.device)
    for w in workers:
        torch.cuda.synchronize(w.device)
    handles = []
    try:
        for w in workers:
            ptrs = (ctypes.c_void_p * 24)()
            present = (ctypes.c_int * 8)()
            for d, r in enumerate(w._peer_neighbours()):
                if r is None:
                    continue
                nb = by_rank[r]
                present[d] = 1
                ptrs[3 * d] = nb.prv.data.data_ptr()      # buffer A = prv now, on every rank
                ptrs[3 * d + 1] = nb.nxt.data.data_ptr()
                ptrs[3 * d + 2] = nb.mailbox.data_ptr()
            hp = ctypes.c_void_p()
            _lib.check(lib.tlb_peer_create_local(w.device.index, ptrs, present,
                                                 ctypes.byref(hp)), "peer create (local)")
            handles.append(hp)
    except ThermoLBError:
        for hp in handles:
            lib.tlb_peer_destroy(hp)
        if strict:
            raise
        return False
    for w, hp in zip(workers, handles):
        with torch.cuda.device(w.device):
            w._adopt_peer(hp, getattr(w.fabric, "timeout", None))
        w.exchange_mode = "p2p"
    return True
