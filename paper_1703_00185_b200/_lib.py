"""ctypes binding of libtlb.so (C ABI declared in include/tlb.h).

This is the only route from Python to the compute: every kernel of the
package is a call into libtlb.so, built in-tree for sm_100a by
``__graft_entry__.build()``.  There is no CPU fallback -- a missing library or
a missing CUDA device raises ``DeviceError``.
"""

import ctypes
import os
import threading

import numpy as np

from .errors import (ContractViolation, DeviceError, DomainError,
                     UnsupportedCaseError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("TLB_LIB_PATH") or os.path.join(HERE, "libtlb.so")

TLB_OK, TLB_ERR_CONTRACT, TLB_ERR_CUDA, TLB_ERR_STENCIL, TLB_ERR_UNSUPPORTED, \
    TLB_ERR_DOMAIN = range(6)

ST_DEGENERATE, ST_SHIFT, ST_EQ_DOMAIN, ST_PEER_TIMEOUT, ST_PROTOCOL = 1, 2, 4, 8, 16

F_WALL_BOT, F_CLAMP_BOT, F_WALL_TOP, F_WRAP_X, F_WRAP_Y, F_COUNT_NEG, F_CLAMP_TOP = \
    1, 4, 2, 8, 16, 32, 64
F_POISON_HALOS = 128
F_CLAMP_Y = F_CLAMP_BOT | F_CLAMP_TOP

ARITH = {"exact": 0, "fast": 1}


class TlbField(ctypes.Structure):
    _fields_ = [("base", ctypes.c_void_p),
                ("sl", ctypes.c_int64), ("sx", ctypes.c_int64), ("sy", ctypes.c_int64),
                ("Lx", ctypes.c_int32), ("Ly", ctypes.c_int32),
                ("Hx", ctypes.c_int32), ("Hy", ctypes.c_int32)]


class TlbParams(ctypes.Structure):
    _fields_ = [("tau", ctypes.c_double), ("gx", ctypes.c_double),
                ("gy", ctypes.c_double), ("dt", ctypes.c_double),
                ("Twall_top", ctypes.c_double), ("Twall_bot", ctypes.c_double),
                ("order", ctypes.c_int32), ("arith", ctypes.c_int32)]


class TlbRegion(ctypes.Structure):
    _fields_ = [("x0", ctypes.c_int32), ("x1", ctypes.c_int32),
                ("y0", ctypes.c_int32), ("y1", ctypes.c_int32)]


class TlbStatus(ctypes.Structure):
    _fields_ = [("flags", ctypes.c_uint32), ("site_x", ctypes.c_int32 * 3),
                ("site_y", ctypes.c_int32 * 3), ("step", ctypes.c_int32),
                ("pad", ctypes.c_uint32), ("negatives", ctypes.c_uint64)]


STATUS_BYTES = ctypes.sizeof(TlbStatus)
STATUS_FLAGS_OFF = TlbStatus.flags.offset
STATUS_NEG_OFF = TlbStatus.negatives.offset

_P = ctypes.c_void_p
_FP = ctypes.POINTER(TlbField)
_PP = ctypes.POINTER(TlbParams)
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_INT = ctypes.c_int

# (name, restype, argtypes) -- mirrors include/tlb.h
SIGNATURES = [
    ("tlb_version", _INT, []),
    ("tlb_last_error", ctypes.c_char_p, []),
    ("tlb_set_device", _INT, [_INT]),
    ("tlb_device_count", _INT, []),
    ("tlb_set_stencil", _INT, [_INT, _P, _P, ctypes.c_double]),
    ("tlb_set_stencil_q", _INT, [_INT, _INT, _P, _P, ctypes.c_double]),
    ("tlb_force_generic", _INT, [_INT, _INT]),
    ("tlb_propagate", _INT, [_FP, _FP, TlbRegion, _P]),
    ("tlb_bc", _INT, [_FP, _PP, _INT, _INT, _I32, _I32, _P, _P]),
    ("tlb_collide", _INT, [_FP, _FP, TlbRegion, _PP, _INT, _P, _P]),
    ("tlb_fused", _INT, [_FP, _FP, TlbRegion, _PP, _INT, _P, _P]),
    ("tlb_step_self", _INT, [_FP, _FP, _PP, _INT, _INT, _INT, _P, _P]),
    ("tlb_step2_self", _INT, [_FP, _FP, _PP, _INT, _INT, _INT, _P, _P, _INT, _P]),
    ("tlb_moments", _INT, [_FP, TlbRegion, _P, _P, _P, _P, _I64, _INT, _P, _P]),
    ("tlb_equilibrium", _INT, [_P, _P, _P, _P, _I64, _INT, _INT, _P, _I64, _INT, _P, _P]),
    ("tlb_apply_shift", _INT, [_P, _P, _P, _I64, _PP, _P, _P, _P, _P, _P]),
    ("tlb_count_negative", _INT, [_FP, TlbRegion, _P, _P]),
    ("tlb_extend_walls", _INT, [_FP, _INT, _INT, _P]),
    ("tlb_face_payload_len", _I64, [_FP]),
    ("tlb_pack_x", _INT, [_FP, _INT, _INT, _P, _P]),
    ("tlb_unpack_x", _INT, [_FP, _INT, _P, _P]),
    ("tlb_face_payload_len_y", _I64, [_FP]),
    ("tlb_pack_y", _INT, [_FP, _INT, _P, _P]),
    ("tlb_unpack_y", _INT, [_FP, _INT, _P, _P]),
    ("tlb_pbc_self_x", _INT, [_FP, _P]),
    ("tlb_pbc_self_y", _INT, [_FP, _P]),
    ("tlb_halo_from_peers", _INT, [_FP, _FP, _FP, _P]),
    ("tlb_nccl_version", _INT, [ctypes.POINTER(_INT)]),
    ("tlb_nccl_unique_id", _INT, [ctypes.c_char_p]),
    ("tlb_ring_create", _INT, [ctypes.c_char_p, _INT, _INT, _INT, ctypes.POINTER(_P)]),
    ("tlb_ring_destroy", _INT, [_P]),
    ("tlb_ring_async_error", _INT, [_P, ctypes.POINTER(_INT)]),
    ("tlb_ring_abort", _INT, [_P]),
    ("tlb_ring_set_neighbors", _INT, [_P, _INT, _INT, _INT, _INT, _P]),
    ("tlb_ring_exchange", _INT, [_P, _FP, _INT, _P, _P, _P]),
    ("tlb_ring_step", _INT, [_P, _FP, _FP, _PP, _INT, _P, _P, _P, _P, _P, _I64, _P]),
    ("tlb_ipc_handle", _INT, [_P, ctypes.c_char_p, ctypes.POINTER(_I64)]),
    ("tlb_peer_create2", _INT, [_INT, ctypes.c_char_p, _P, _P, ctypes.POINTER(_P)]),
    ("tlb_peer_destroy", _INT, [_P]),
    ("tlb_peer_create_local", _INT, [_INT, _P, _P, ctypes.POINTER(_P)]),
    ("tlb_peer_set_timeout", _INT, [_P, ctypes.c_double]),
    ("tlb_peer_step", _INT, [_P, _FP, _FP, _INT, _PP, _INT, _P, _P, _I64, _I64, _INT, _P]),
    ("tlb_peer_prime", _INT, [_P, _FP, _INT, _PP, _P, _P, _I64, _I64, _P]),
    ("tlb_peer_step2", _INT, [_P, _FP, _FP, _INT, _PP, _INT, _P, _P, _P, _I64, _I64, _INT, _P]),
    ("tlb_peer_prime2", _INT, [_P, _FP, _INT, _PP, _P, _P, _I64, _I64, _P]),
    ("tlb_pgm_image", _INT, [_P, _I64, _I64, _I64, _P, _P, _P]),
    ("tlb_set_tuning", _INT, [_INT, _INT]),
    ("tlb_get_tuning", _INT, [_INT, ctypes.POINTER(ctypes.c_int)]),
    ("tlb_bench_dfma", _INT, [_I64, ctypes.POINTER(ctypes.c_double), _P]),
]

_lib = None
_lock = threading.Lock()
_stencil_devices = {}


def load():
    """Load libtlb.so (no GPU needed to load; every export is bound)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise DeviceError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -c 'import __graft_entry__ as g; g.build()'` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(LIB_PATH)
            for name, res, args in SIGNATURES:
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error():
    return load().tlb_last_error().decode(errors="replace")


def check(code, what=""):
    if code == TLB_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if code == TLB_ERR_CONTRACT:
        raise ContractViolation(msg)
    if code == TLB_ERR_DOMAIN:
        raise DomainError(msg)
    if code == TLB_ERR_UNSUPPORTED or code == TLB_ERR_STENCIL:
        raise UnsupportedCaseError(msg)
    raise DeviceError(msg)


def torch_cuda():
    """torch, with a CUDA device required (no CPU fallback)."""
    import torch
    if not torch.cuda.is_available():
        raise DeviceError("no CUDA device: the D2Q37 kernels run only on the GPU "
                          "(sm_100a); there is no CPU fallback")
    return torch


def ensure_stencil(vs, device):
    """Upload vs's constants to `device` when they change (tlb_set_stencil_q):
    the reference D2Q37 ordering runs the specialised kernels, other stencils
    (D2Q9) the generic ones."""
    key = (int(device), vs.c.tobytes(), vs.w.tobytes(), float(vs.cs2))
    if _stencil_devices.get(int(device)) == key:
        return
    lib = load()
    c = np.ascontiguousarray(vs.c, dtype=np.int64)
    w = np.ascontiguousarray(vs.w, dtype=np.float64)
    check(lib.tlb_set_stencil_q(int(device), int(vs.Q), c.ctypes.data, w.ctypes.data,
                                float(vs.cs2)), "set_stencil")
    _stencil_devices[int(device)] = key


def field(t, Lx=None, Ly=None, H=0, Hy=None):
    """TlbField over a torch float64 CUDA tensor viewed as (Q, NX, NY)."""
    import torch
    if t.dtype != torch.float64 or not t.is_cuda:
        raise ContractViolation("fields must be float64 CUDA tensors")
    if t.dim() != 3:
        raise ContractViolation(f"expected a (Q, NX, NY) view, got shape {tuple(t.shape)}")
    Hx = H
    Hy = H if Hy is None else Hy
    if Lx is None:
        Lx = t.shape[1] - 2 * Hx
    if Ly is None:
        Ly = t.shape[2] - 2 * Hy
    sl, sx, sy = t.stride()
    return TlbField(t.data_ptr(), sl, sx, sy, Lx, Ly, Hx, Hy)


def params(p, vs=None):
    """TlbParams from a PhysicsParams; eq_order None means the stencil's own
    order (kernels.py:80-81: 4 for D2Q37, 2 for D2Q9)."""
    order = p.eq_order if p.eq_order is not None else (vs.eq_order if vs is not None else 4)
    arith = ARITH.get(getattr(p, "arith", "exact"))
    if arith is None:
        raise DomainError(f"unknown arith mode {p.arith!r}")
    return TlbParams(p.tau, p.gx, p.gy, p.dt, p.Twall_top, p.Twall_bot, order, arith)


def region(x0, x1, y0, y1):
    return TlbRegion(int(x0), int(x1), int(y0), int(y1))


def stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Status:
    """Device-resident TlbStatus block plus host-side decoding."""

    def __init__(self, device):
        import torch
        self.buf = torch.zeros(STATUS_BYTES, dtype=torch.uint8, device=device)

    @property
    def ptr(self):
        return self.buf.data_ptr()

    def reset(self):
        self.buf.zero_()

    def read(self):
        raw = bytes(self.buf.cpu().numpy())
        return TlbStatus.from_buffer_copy(raw)
