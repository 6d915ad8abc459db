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
  pbc, propagate, bc, collide) -- bitwise the reference, 1184 B/site;
  schedule "overlapped" is the B200 path: one fused propagate+bc+collide
  kernel per region with the wall extension and (for a single rank) the
  periodic X wrap folded into its loads, the X-face exchange overlapped with
  the bulk columns on a side stream, then the 3+3 border columns -- 592 B/site.

2-D tilings (Y exchange, pbc_nc between ranks) are outside this round's
scope: ``RankWorker`` raises UnsupportedCaseError for them.
"""

import math
import queue
import threading
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import (ConfigurationError, DeadlockError, DegenerateStateError,
                     DomainError, ProtocolError, ThermoLBError,
                     UnsupportedCaseError)
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
    """Split the lattice into Np uniform tiles (runtime.py:54-91)."""
    if tiling == "1d":
        nx, ny = Np, 1
    else:
        nx, ny = tiling
    if nx * ny != Np:
        raise ConfigurationError(f"grid {nx}x{ny} does not match Np={Np}")
    if Lx % nx:
        raise ConfigurationError(f"Lx={Lx} not divisible by nx={nx}; " + _divisor_hint(Lx, "X"))
    if Ly % ny:
        raise ConfigurationError(f"Ly={Ly} not divisible by ny={ny}; " + _divisor_hint(Ly, "Y"))
    tx, ty = Lx // nx, Ly // ny
    tiles = []
    for iy in range(ny):
        for ix in range(nx):
            rank = iy * nx + ix
            left = iy * nx + (ix - 1) % nx
            right = iy * nx + (ix + 1) % nx
            if periodic_y:
                up = ((iy + 1) % ny) * nx + ix
                down = ((iy - 1) % ny) * nx + ix
            else:
                up = (iy + 1) * nx + ix if iy + 1 < ny else None
                down = (iy - 1) * nx + ix if iy > 0 else None
            tiles.append(TileAssignment(
                rank=rank, grid=(nx, ny), coords=(ix, iy), Lx=tx, Ly=ty,
                x0=ix * tx, y0=iy * ty,
                neighbors={"left": left, "right": right, "up": up, "down": down},
                uppermost=(not periodic_y) and iy == ny - 1,
                lowermost=(not periodic_y) and iy == 0))
    return tiles


def face_plans(vs: VelocitySet, depth=DEFAULT_HALO):
    """plans[(axis, sign)][d-1] = indices l with sign * c_l[axis] >= d
    (runtime.py:94-107)."""
    plans = {}
    for axis in (0, 1):
        for sign in (1, -1):
            plans[(axis, sign)] = [np.nonzero(sign * vs.c[:, axis] >= d)[0]
                                   for d in range(1, depth + 1)]
    return plans


def boundary_bytes_per_site(vs: VelocitySet, depth=DEFAULT_HALO):
    """Bytes crossing one face per boundary site (runtime.py:110-113)."""
    return 8 * sum(len(ls) for ls in face_plans(vs, depth)[(0, 1)])


# --------------------------------------------------------------- fabrics --

class Fabric:
    """In-process point-to-point channels with the reference's semantics
    (runtime.py:116-160): ordered, tagged with the step, recv times out with
    DeadlockError naming the stalled rank, a step mismatch is a
    ProtocolError.  Payloads are device tensors; the sender attaches a CUDA
    event so the receiver's stream waits for the pack without a host sync."""

    def __init__(self, Np, timeout=60.0):
        self.Np = Np
        self.timeout = timeout
        self.channels = {}
        self.abort = threading.Event()
        self.failures = []
        self._lock = threading.Lock()

    def _chan(self, src, dst, tag):
        key = (src, dst, tag)
        with self._lock:
            if key not in self.channels:
                self.channels[key] = queue.Queue()
            return self.channels[key]

    def send(self, src, dst, tag, step, payload, event=None):
        self._chan(src, dst, tag).put((step, payload, event))

    def recv(self, dst, src, tag, step, with_event=False):
        chan = self._chan(src, dst, tag)
        deadline = time.monotonic() + self.timeout
        while True:
            if self.abort.is_set():
                raise ThermoLBError(f"rank {dst}: aborted by peer failure")
            try:
                got_step, payload, event = chan.get(timeout=min(_POLL, self.timeout))
            except queue.Empty:
                if time.monotonic() > deadline:
                    raise DeadlockError(
                        f"rank {dst} stalled waiting for rank {src} (tag {tag}, step {step})",
                        rank=dst)
                continue
            if got_step != step:
                raise ProtocolError(
                    f"rank {dst}: expected step {step} from {src}/{tag}, got {got_step}")
            return (payload, event) if with_event else payload

    def fail(self, rank, exc):
        with self._lock:
            self.failures.append((rank, exc))
        self.abort.set()

    # -- X-face exchange used by RankWorker -------------------------------
    def start_x(self, w, step, out_plus, out_minus):
        torch = _lib.torch_cuda()
        ev = torch.cuda.Event()
        ev.record(w.stream)
        nb = w.tile.neighbors
        self.send(w.tile.rank, nb["right"], "x+", step, out_plus, ev)
        self.send(w.tile.rank, nb["left"], "x-", step, out_minus, ev)
        return step

    def finish_x(self, w, handle, in_plus, in_minus, stream=None):
        torch = _lib.torch_cuda()
        stream = stream or w.stream
        step = handle
        nb = w.tile.neighbors
        for tag, src, dst in (("x+", nb["left"], in_plus), ("x-", nb["right"], in_minus)):
            payload, ev = self.recv(w.tile.rank, src, tag, step, with_event=True)
            if payload.numel() != dst.numel():
                raise ProtocolError(f"rank {w.tile.rank}: X payload size mismatch")
            if ev is not None:
                stream.wait_event(ev)
            with torch.cuda.stream(stream):
                dst.copy_(payload, non_blocking=True)
            if payload.device == dst.device:
                payload.record_stream(stream)
            else:
                w.retain(payload)  # peer copy: keep alive until the next sync


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

    def start_x(self, w, step, out_plus, out_minus):
        dist = self.dist
        nb = w.tile.neighbors
        ops = [dist.P2POp(dist.isend, out_plus, nb["right"], self.group),
               dist.P2POp(dist.isend, out_minus, nb["left"], self.group),
               dist.P2POp(dist.irecv, w.rbuf_plus, nb["left"], self.group),
               dist.P2POp(dist.irecv, w.rbuf_minus, nb["right"], self.group)]
        return dist.batch_isend_irecv(ops)

    def finish_x(self, w, handle, in_plus, in_minus, stream=None):
        # called under torch.cuda.stream(stream): wait() orders it after NCCL
        for req in handle:
            try:
                req.wait()
            except Exception as exc:  # timeouts surface as DeadlockError
                raise DeadlockError(f"rank {w.tile.rank} stalled in the X exchange: {exc}",
                                    rank=w.tile.rank) from exc

    def fail(self, rank, exc):
        self.failures.append((rank, exc))
        self.abort.set()


# ------------------------------------------------------------ rank worker --

@dataclass
class _StepRecord:
    step: int
    status: object      # device slice (bytes) of the per-step status ring
    events: tuple       # (t0, t1, t2, t3) CUDA events: comm / bulk / border


class RankWorker:
    """One rank: owns a tile's double buffer in HBM and runs the step loop
    (runtime.py:163-404).

    ``fabric`` is a ``Fabric`` (in-process ranks) or ``DistFabric`` (one
    process per GPU).  ``device`` selects the GPU (default: current)."""

    def __init__(self, tile, vs, params, fabric=None, schedule="staged", walls=True,
                 layout="soa", halo=DEFAULT_HALO, debug_poison=False, device=None,
                 periodic_y=False):
        torch = _lib.torch_cuda()
        if tile.grid[1] != 1:
            raise UnsupportedCaseError(
                "2-D tilings (Y exchange between ranks) are not built in this round; "
                "use tiling='1d'")
        if schedule not in ("staged", "overlapped"):
            raise ConfigurationError(f"unknown schedule {schedule!r}")
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
        self.geom = LatticeGeometry(tile.Lx, tile.Ly, halo, halo, vs.Q, layout)
        self.halo = halo
        with torch.cuda.device(self.device):
            _lib.ensure_stencil(vs, self.device.index)
            self.prv, self.nxt = allocate_field(self.geom, vs, device=self.device)
            self.stream = torch.cuda.Stream(self.device)
            self.comm_stream = torch.cuda.Stream(self.device, priority=-1)
            n = int(_lib.load().tlb_face_payload_len(field_desc(self.prv)))
            self.payload_len = n
            self.rbuf_plus = torch.empty(n, dtype=torch.float64, device=self.device)
            self.rbuf_minus = torch.empty(n, dtype=torch.float64, device=self.device)
            self._ring = None
            if isinstance(fabric, DistFabric) and fabric.native and tile.grid[0] > 1:
                self._ring = fabric.ring(self.device.index)
                self.sbuf2 = torch.empty(2 * n, dtype=torch.float64, device=self.device)
                self.rbuf2 = torch.empty(2 * n, dtype=torch.float64, device=self.device)
            self._status_ring = torch.zeros((self._RING, _lib.STATUS_BYTES),
                                            dtype=torch.uint8, device=self.device)
            # order the allocations' zero-fills before any work on our stream
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
        self.plans = face_plans(vs, halo)
        self.tparams = _lib.params(params)
        self._records = []
        self._retained = []
        self._metrics = []
        self.snapshots = []

    # -- helpers -------------------------------------------------------------
    @property
    def Np(self):
        return self.tile.grid[0]

    @property
    def self_ring(self):
        return self.tile.neighbors["left"] == self.tile.rank

    def _sp(self):
        return self.stream.cuda_stream

    def _check(self, code, what):
        _lib.check(code, what)

    def _wall_flags(self):
        f = 0
        if self.walls and self.tile.lowermost:
            f |= _lib.F_WALL_BOT
        if self.walls and self.tile.uppermost:
            f |= _lib.F_WALL_TOP
        return f

    def _ymode(self):
        if self.walls:
            return 1
        if self.periodic_y:
            return 2
        return 0

    _RING = 1024

    def _status_slot(self):
        if len(self._records) >= self._RING:
            self.collect()
        return self._status_ring[len(self._records)]

    def retain(self, t):
        self._retained.append(t)

    # -- halo exchange (reference names) -------------------------------------
    def pack_x(self, f, sign, ymode=0):
        """Outgoing X-face payload (runtime.py:199-208); a new device tensor."""
        torch = _lib.torch_cuda()
        with torch.cuda.stream(self.stream):
            buf = torch.empty(self.payload_len, dtype=torch.float64, device=self.device)
        self._check(_lib.load().tlb_pack_x(field_desc(f), int(sign), int(ymode),
                                           buf.data_ptr(), self._sp()), "pack_x")
        return buf

    def unpack_x(self, f, sign, payload, stream=None):
        """Scatter a received X payload into the halo columns (runtime.py:210-224)."""
        torch = _lib.torch_cuda()
        if not isinstance(payload, torch.Tensor):
            payload = torch.as_tensor(np.asarray(payload, dtype=np.float64), device=self.device)
        if payload.numel() != self.payload_len:
            raise ProtocolError(f"rank {self.tile.rank}: X payload size mismatch")
        sp = (stream or self.stream).cuda_stream
        self._check(_lib.load().tlb_unpack_x(field_desc(f), int(sign), payload.data_ptr(),
                                             sp), "unpack_x")

    def pbc_c(self, f, step):
        """Exchange the X halo columns around the ring (runtime.py:281-284)."""
        if self.self_ring:
            self._check(_lib.load().tlb_pbc_self_x(field_desc(f), self._sp()), "pbc_c")
            return
        h = self._start_exchange(step, self.pack_x(f, 1), self.pack_x(f, -1))
        self._finish_exchange(f, h)

    def _start_exchange(self, step, out_plus, out_minus):
        torch = _lib.torch_cuda()
        with torch.cuda.stream(self.stream):
            return self.fabric.start_x(self, step, out_plus, out_minus)

    def _finish_exchange(self, f, handle, stream=None):
        torch = _lib.torch_cuda()
        stream = stream or self.stream
        with torch.cuda.stream(stream):
            self.fabric.finish_x(self, handle, self.rbuf_plus, self.rbuf_minus, stream)
        self.unpack_x(f, 1, self.rbuf_plus, stream)
        self.unpack_x(f, -1, self.rbuf_minus, stream)

    def _extend_wall_halos(self, f):
        """runtime.py:296-305."""
        up = self.walls and self.tile.uppermost
        lo = self.walls and self.tile.lowermost
        if up or lo:
            self._check(_lib.load().tlb_extend_walls(field_desc(f), int(up), int(lo),
                                                     self._sp()), "extend_walls")

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
        if self.walls and self.tile.lowermost:
            rows.append((g.Hy, g.Hy + WALL_ROWS))
        if self.walls and self.tile.uppermost:
            rows.append((g.Hy + g.Ly - WALL_ROWS, g.Hy + g.Ly))
        return rows

    # -- schedules -----------------------------------------------------------
    def _fused(self, x0, x1, flags, st, stream=None):
        g = self.geom
        if x1 <= x0:
            return
        sp = (stream or self.stream).cuda_stream
        self._check(_lib.load().tlb_fused(
            field_desc(self.prv), field_desc(self.nxt),
            _lib.region(x0, x1, g.Hy, g.Hy + g.Ly), self.tparams, flags, st, sp), "fused")

    def step(self, step_no):
        """One time step (runtime.py:355-400), enqueued on the rank's stream."""
        self.step_begin(step_no)
        self.step_end(step_no)

    def step_begin(self, step_no):
        torch = _lib.torch_cuda()
        g = self.geom
        lib = _lib.load()
        slot = self._status_slot()
        st = slot.data_ptr()
        ev = tuple(torch.cuda.Event(enable_timing=True) for _ in range(4))
        self._pending = (step_no, slot, ev, st)
        ev[0].record(self.stream)
        if self.debug_poison:
            self._poison_halos(self.prv)
        if self.schedule == "staged":
            # reference path, op for op
            if self.walls:
                self._extend_wall_halos(self.prv)
            if self.periodic_y:
                self._check(lib.tlb_pbc_self_y(field_desc(self.prv), self._sp()), "pbc_nc")
            if self.self_ring:
                self._check(lib.tlb_pbc_self_x(field_desc(self.prv), self._sp()), "pbc_c")
                self._handle = None
            elif self._ring is not None:
                self._check(lib.tlb_ring_exchange(
                    self._ring, field_desc(self.prv), 0, self.sbuf2.data_ptr(),
                    self.rbuf2.data_ptr(), self._sp()), "ring exchange")
                self._handle = None
            else:
                self._handle = self._start_exchange(step_no, self.pack_x(self.prv, 1),
                                                    self.pack_x(self.prv, -1))
            ev[1].record(self.stream)
            return
        # overlapped: fused kernels with the wall extension folded in
        flags = self._wall_flags() | _lib.F_COUNT_NEG
        if self.walls:
            flags |= _lib.F_CLAMP_Y
        elif self.periodic_y:
            flags |= _lib.F_WRAP_Y
        self._flags = flags
        if self.self_ring:
            ev[1].record(self.stream)
            self._check(lib.tlb_fused(
                field_desc(self.prv), field_desc(self.nxt),
                _lib.region(g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly), self.tparams,
                flags | _lib.F_WRAP_X, st, self._sp()), "fused")
            self._handle = None
            return
        if self._ring is not None:
            ev[1].record(self.stream)
            ev[2].record(self.stream)
            self._check(lib.tlb_ring_step(
                self._ring, field_desc(self.prv), field_desc(self.nxt), self.tparams, flags,
                st, self.sbuf2.data_ptr(), self.rbuf2.data_ptr(), ev[1].cuda_event,
                ev[2].cuda_event, self._sp()), "ring step")
            self._handle = None
            return
        h = self.halo
        ymode = self._ymode()
        out_p = self.pack_x(self.prv, 1, ymode)
        out_m = self.pack_x(self.prv, -1, ymode)
        self._handle = self._start_exchange(step_no, out_p, out_m)
        ev[1].record(self.stream)
        self._fused(g.Hx + h, g.Hx + g.Lx - h, flags, st)   # bulk columns
        ev[2].record(self.stream)

    def step_end(self, step_no):
        g = self.geom
        lib = _lib.load()
        step_no_, slot, ev, st = self._pending
        if self.schedule == "staged":
            if self._handle is not None:
                self._finish_exchange(self.prv, self._handle)
            ev[2].record(self.stream)
            full = _lib.region(g.Hx, g.Hx + g.Lx, g.Hy, g.Hy + g.Ly)
            self._check(lib.tlb_propagate(field_desc(self.prv), field_desc(self.nxt), full,
                                          self._sp()), "propagate")
            if self.walls and (self.tile.uppermost or self.tile.lowermost):
                self._check(lib.tlb_bc(field_desc(self.nxt), self.tparams,
                                       int(self.tile.uppermost), int(self.tile.lowermost),
                                       g.Hx, g.Hx + g.Lx, st, self._sp()), "bc")
            self._check(lib.tlb_collide(field_desc(self.nxt), field_desc(self.nxt), full,
                                        self.tparams, _lib.F_COUNT_NEG, st, self._sp()),
                        "collide")
        else:
            if self._handle is not None:
                # halo arrival -> unpack -> 3+3 border columns on the
                # high-priority side stream, concurrent with the bulk kernel
                cs = self.comm_stream
                self._finish_exchange(self.prv, self._handle, cs)
                h = self.halo
                self._fused(g.Hx, g.Hx + h, self._flags, st, cs)
                self._fused(g.Hx + g.Lx - h, g.Hx + g.Lx, self._flags, st, cs)
                self.stream.wait_stream(cs)
            elif self._ring is None:
                ev[2].record(self.stream)
        ev[3].record(self.stream)
        self._records.append(_StepRecord(step_no, slot, ev))
        self.prv, self.nxt = swap_buffers(self.prv, self.nxt)

    # -- results -------------------------------------------------------------
    def synchronize(self):
        self.stream.synchronize()

    def collect(self, raise_errors=True):
        """Materialise pending per-step metrics (one host sync) and raise the
        first per-site failure the kernels flagged, like the reference's
        in-step exceptions (kernels.py:62-66, 134-135, 85-86)."""
        if not self._records:
            return
        self.synchronize()
        n = len(self._records)
        raw = self._status_ring[:n].cpu().numpy()
        err = None
        for rec, row in zip(self._records, raw):
            s = _lib.TlbStatus.from_buffer_copy(row.tobytes())
            t0, t1, t2, t3 = rec.events
            if self.schedule == "staged":
                m = {"t_comm_nc": 0.0, "t_comm_c": t0.elapsed_time(t2) * 1e-3,
                     "t_bulk": t2.elapsed_time(t3) * 1e-3, "t_border": 0.0}
            else:
                m = {"t_comm_nc": 0.0, "t_comm_c": t0.elapsed_time(t1) * 1e-3,
                     "t_bulk": t1.elapsed_time(t2) * 1e-3,
                     "t_border": t2.elapsed_time(t3) * 1e-3}
            m["negatives"] = int(s.negatives)
            self._metrics.append(m)
            if err is None and s.flags:
                err = (rec.step, s)
        self._records = []
        self._retained = []
        with _lib.torch_cuda().cuda.stream(self.stream):
            self._status_ring.zero_()
        if err is not None and raise_errors:
            step, s = err
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
        g = self.geom
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(self.stream):
            src = block if isinstance(block, torch.Tensor) else torch.as_tensor(
                np.ascontiguousarray(block, dtype=np.float64))
            self.prv.pops[:, g.phys_x, g.phys_y].copy_(src, non_blocking=True)
            if src.is_cuda and src.device == self.device:
                src.record_stream(self.stream)
