"""ctypes front-end of the C oracle (``tlb_oracle.c``) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) import this module, and only
as the checker / CPU baseline.  The product package never imports it.

The functions take and return numpy arrays in the reference's canonical
layout (``(Q, NX, NY)`` fields, ``(Q, n)`` blocks) and mirror the signatures
of ``thermolb.kernels`` (``/root/reference/pkg/src/thermolb/kernels.py``).
Initial-condition macro fields are restated in numpy from ``init.py:14-64``.
"""

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libtlb_oracle.so")

_P = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64
_lib = None


def build():
    """Compile the oracle with its committed Makefile (gcc, no FMA)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.orc_set_stencil.argtypes = [ctypes.POINTER(_I64), _P, ctypes.c_double]
        L.orc_last_error.argtypes = [ctypes.POINTER(_I64)]
        L.orc_moments.argtypes = [_P, _I64, _I64, _P, _P, _P, _P, ctypes.c_int]
        L.orc_equilibrium.argtypes = [_P, _P, _P, _P, _I64, ctypes.c_int, _P,
                                      _I64, ctypes.c_int]
        L.orc_collide.argtypes = [_P, _P, _I64, _I64, _I64, _P, ctypes.c_int]
        L.orc_propagate.argtypes = [_P, _P] + [_I64] * 7
        L.orc_bc.argtypes = [_P] + [_I64] * 5 + [ctypes.c_int, ctypes.c_int,
                                                 _P, ctypes.c_int]
        L.orc_collide_region.argtypes = [_P] + [_I64] * 7 + [_P, ctypes.c_int]
        L.orc_fused.argtypes = [_P, _P] + [_I64] * 7 + [_P, ctypes.c_int]
        L.orc_extend_walls.argtypes = [_P, _I64, _I64, _I64, ctypes.c_int,
                                       ctypes.c_int]
        L.orc_pbc_self.argtypes = [_P, _I64, _I64, _I64]
        L.orc_pbc_y_self.argtypes = [_P, _I64, _I64, _I64]
        L.orc_count_negative.argtypes = [_P, _I64, _I64, _I64]
        L.orc_count_negative.restype = _I64
        L.orc_step.argtypes = [_P, _P, _I64, _I64, _I64, ctypes.c_int, _P,
                               ctypes.c_int, ctypes.POINTER(_I64)]
        L.orc_run.argtypes = [_P, _P, _I64, _I64, _I64, _I64, ctypes.c_int, _P,
                              ctypes.c_int, ctypes.POINTER(_I64)]
        L.orc_run_timed.argtypes = [_P, _P, _I64, _I64, _I64, _I64, _I64, ctypes.c_int, _P,
                                    ctypes.c_int, ctypes.POINTER(ctypes.c_double)]
        L.orc_set_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _ptr(a):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_P)


class OracleError(RuntimeError):
    """Raised with the oracle's error code (1 degenerate rho, 2 T_bar<=0,
    3 bc/equilibrium domain, 4 region contract, 5 allocation)."""

    def __init__(self, code, site=-1):
        super().__init__(f"oracle error {code} at site {site}")
        self.code, self.site = code, site


def _check(code):
    if code:
        site = _I64(-1)
        lib().orc_last_error(ctypes.byref(site))
        raise OracleError(code, site.value)


def set_stencil(c, w, cs2):
    c = np.ascontiguousarray(c, dtype=np.int64)
    w = np.ascontiguousarray(w, dtype=np.float64)
    assert c.shape == (37, 2) and w.shape == (37,)
    lib().orc_set_stencil(c.ctypes.data_as(ctypes.POINTER(_I64)), _ptr(w),
                          float(cs2))


def params6(tau, gx=0.0, gy=0.0, dt=1.0, Twall_top=1.0, Twall_bot=1.0):
    return np.array([tau, gx, gy, dt, Twall_top, Twall_bot], dtype=np.float64)


def threads(n):
    lib().orc_set_threads(int(n))


# ---- block API -------------------------------------------------------------

def moments(f, check=True):
    f = np.ascontiguousarray(f, dtype=np.float64)
    shape = f.shape[1:]
    f2 = f.reshape(37, -1)
    n = f2.shape[1]
    out = [np.empty(n) for _ in range(4)]
    _check(lib().orc_moments(_ptr(f2), n, n, *[_ptr(o) for o in out],
                             int(check)))
    return tuple(o.reshape(shape) for o in out)


def equilibrium(rho, ux, uy, T, order=4, check=True):
    arrs = np.broadcast_arrays(*[np.asarray(a, dtype=np.float64)
                                 for a in (rho, ux, uy, T)])
    shape = arrs[0].shape
    flat = [np.ascontiguousarray(a).reshape(-1) for a in arrs]
    n = flat[0].size
    out = np.empty((37, n))
    _check(lib().orc_equilibrium(*[_ptr(a) for a in flat], n, order,
                                 _ptr(out), n, int(check)))
    return out.reshape((37,) + shape)


def collide(f, p6, order=4):
    f = np.ascontiguousarray(f, dtype=np.float64)
    shape = f.shape
    f2 = f.reshape(37, -1)
    n = f2.shape[1]
    out = np.empty_like(f2)
    _check(lib().orc_collide(_ptr(f2), _ptr(out), n, n, n, _ptr(p6), order))
    return out.reshape(shape)


# ---- field API (canonical (Q, NX, NY), halo H) -----------------------------

def _dims(field, H):
    Q, NX, NY = field.shape
    return NX - 2 * H, NY - 2 * H


def propagate(prv, nxt, H, region=None):
    Lx, Ly = _dims(prv, H)
    x0, x1, y0, y1 = region or (H, H + Lx, H, H + Ly)
    _check(lib().orc_propagate(_ptr(prv), _ptr(nxt), Lx, Ly, H, x0, x1, y0, y1))


def bc(field, H, p6, top=True, bottom=True, x_range=None, order=4):
    Lx, Ly = _dims(field, H)
    x0, x1 = x_range or (H, H + Lx)
    _check(lib().orc_bc(_ptr(field), Lx, Ly, H, x0, x1, int(top), int(bottom),
                        _ptr(p6), order))


def collide_region(field, H, p6, region=None, order=4):
    Lx, Ly = _dims(field, H)
    x0, x1, y0, y1 = region or (H, H + Lx, H, H + Ly)
    _check(lib().orc_collide_region(_ptr(field), Lx, Ly, H, x0, x1, y0, y1,
                                    _ptr(p6), order))


def fused(prv, nxt, H, p6, region=None, order=4):
    Lx, Ly = _dims(prv, H)
    x0, x1, y0, y1 = region or (H, H + Lx, H, H + Ly)
    _check(lib().orc_fused(_ptr(prv), _ptr(nxt), Lx, Ly, H, x0, x1, y0, y1,
                           _ptr(p6), order))


def extend_walls(field, H, upper=True, lower=True):
    Lx, Ly = _dims(field, H)
    lib().orc_extend_walls(_ptr(field), Lx, Ly, H, int(upper), int(lower))


def pbc_self(field, H):
    Lx, Ly = _dims(field, H)
    lib().orc_pbc_self(_ptr(field), Lx, Ly, H)


def count_negative(field, H):
    Lx, Ly = _dims(field, H)
    return int(lib().orc_count_negative(_ptr(field), Lx, Ly, H))


YMODES = {"walls": 1, "periodic": 2, "none": 0}


def run(f0, steps, p6, H=3, ymode="walls", order=4, nthreads=None):
    """Np=1 run (sim.py:62-129): f0 is the (Q, Lx, Ly) physical block.
    Returns (final block, per-step negatives)."""
    if nthreads:
        threads(nthreads)
    f0 = np.ascontiguousarray(f0, dtype=np.float64)
    _, Lx, Ly = f0.shape
    out = np.empty_like(f0)
    neg = np.zeros(max(steps, 1), dtype=np.int64)
    _check(lib().orc_run(_ptr(f0), _ptr(out), Lx, Ly, H, steps, YMODES[ymode],
                         _ptr(p6), order,
                         neg.ctypes.data_as(ctypes.POINTER(_I64))))
    return out, neg[:steps]


def run_timed(f0, warmup, steps, p6, H=3, ymode="walls", order=4):
    """bench.py's CPU leg: `warmup` untimed steps, then `steps` steps timed
    inside the C library (monotonic clock).  Returns (final block, seconds)."""
    f0 = np.ascontiguousarray(f0, dtype=np.float64)
    _, Lx, Ly = f0.shape
    out = np.empty_like(f0)
    sec = ctypes.c_double(0.0)
    _check(lib().orc_run_timed(_ptr(f0), _ptr(out), Lx, Ly, H, warmup, steps, YMODES[ymode],
                               _ptr(p6), order, ctypes.byref(sec)))
    return out, sec.value


# ---- initial conditions (numpy restatement of init.py) ---------------------

def rayleigh_taylor_macro(Lx, Ly, cs2, T_hot=None, T_cold=None,
                          perturbation=0.02, width=2.0):
    """(rho, ux, uy, T) handed to equilibrium by init.rayleigh_taylor
    (init.py:45-64)."""
    if T_hot is None:
        T_hot = cs2 * 1.1
    if T_cold is None:
        T_cold = cs2 * 0.9
    x = np.arange(Lx)[:, None] + 0.5
    y = np.arange(Ly)[None, :] + 0.5
    interface = Ly / 2.0 + perturbation * Ly * np.cos(2.0 * np.pi * x / Lx)
    frac = 0.5 * (1.0 + np.tanh((y - interface) / width))
    T = T_hot + (T_cold - T_hot) * frac
    p0 = T_hot
    rho = p0 / T
    z = np.zeros((Lx, Ly))
    return rho, z, z, T * np.ones((Lx, Ly))


def random_near_equilibrium_macro(Lx, Ly, cs2, seed=0, amplitude=0.01):
    """init.py:22-30."""
    rng = np.random.default_rng(seed)
    shape = (Lx, Ly)
    rho = 1.0 + amplitude * rng.standard_normal(shape)
    ux = amplitude * rng.standard_normal(shape)
    uy = amplitude * rng.standard_normal(shape)
    T = cs2 * (1.0 + amplitude * rng.standard_normal(shape))
    return rho, ux, uy, T


def pad(block, H=3):
    """Place a (Q, Lx, Ly) block into a zeroed (Q, NX, NY) field."""
    Q, Lx, Ly = block.shape
    f = np.zeros((Q, Lx + 2 * H, Ly + 2 * H))
    f[:, H:H + Lx, H:H + Ly] = block
    return f
