"""The three computational kernels -- propagate (pull), bc, collide -- plus
the fused variant, moments, equilibrium and the monitors, on the GPU.

Drop-in for kernels.py of the reference (/root/reference/pkg/src/thermolb/
kernels.py): same names, signatures, argument meaning, ownership and
exceptions.  Fields are ``PopulationField`` objects whose ``.pops`` is the
canonical (Q, NX, NY) view (here a float64 CUDA tensor); ``region`` is a
(slice_x, slice_y) pair in padded coordinates.  Block functions (collide,
moments, equilibrium) accept torch CUDA tensors (results stay on the device)
or numpy arrays (uploaded, computed by the same CUDA kernels, returned as
numpy).  Every computation is a call into libtlb.so (include/tlb.h); there is
no CPU fallback.

Arithmetic: ``PhysicsParams.arith = "exact"`` (default) reproduces the
reference bit for bit; ``"fast"`` uses FMA and a regrouped polynomial
(~1e-15 relative per step; see csrc/d2q37.cuh).
"""

from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ContractViolation, DegenerateStateError, DomainError
from .geometry import LatticeGeometry, PopulationField
from .velocity_set import VelocitySet

WALL_ROWS = 3  # kernels.py:18


@dataclass(frozen=True)
class PhysicsParams:
    """Relaxation time, body force and wall temperatures (kernels.py:21-38).

    ``arith`` selects the collide arithmetic: "exact" (bitwise equal to the
    reference) or "fast" (FMA-contracted, ~1e-15 relative per step)."""

    tau: float
    gx: float = 0.0
    gy: float = 0.0
    dt: float = 1.0
    D: int = 2
    Twall_top: float = 1.0
    Twall_bot: float = 1.0
    eq_order: int | None = None
    arith: str = "exact"

    def __post_init__(self):
        if self.tau <= self.dt / 2:
            raise DomainError(f"tau={self.tau} violates tau > dt/2")
        if self.D != 2:
            raise DomainError("only D=2 is supported")
        if self.arith not in _lib.ARITH:
            raise DomainError(f"unknown arith mode {self.arith!r} (exact|fast)")


# ------------------------------------------------------------------ helpers --

_status_cache = {}


def _status(device):
    key = str(device)
    st = _status_cache.get(key)
    if st is None:
        st = _status_cache[key] = _lib.Status(device)
    return st


def _to_device(a, like=None):
    """(tensor, numpy_in) -- numpy/scalars are uploaded to the current device."""
    torch = _lib.torch_cuda()
    if isinstance(a, torch.Tensor):
        if not a.is_cuda:
            a = a.cuda()
        return a.to(torch.float64), False
    dev = like.device if like is not None else torch.device("cuda", torch.cuda.current_device())
    return torch.as_tensor(np.array(a, dtype=np.float64), device=dev), True


def _block3(t):
    """A (Q, ...) tensor as a (Q, a, b) strided view for a halo-free field."""
    if t.dim() == 1:
        return t.view(t.shape[0], 1, 1)
    if t.dim() == 2:
        return t.unsqueeze(1)
    if t.dim() == 3:
        return t
    return t.reshape(t.shape[0], -1, t.shape[-1])


def _out(t, numpy_in):
    return t.cpu().numpy() if numpy_in else t


def _vs_device(vs, t):
    _lib.ensure_stencil(vs, t.device.index or 0)


def _raise_status(st, what):
    s = st.read()
    if s.flags & _lib.ST_EQ_DOMAIN:
        raise DomainError("equilibrium requires rho > 0 and T > 0")
    if s.flags & _lib.ST_DEGENERATE:
        site = (s.site_x[0], s.site_y[0])
        raise DegenerateStateError(f"non-positive density at {[list(site)]} ({what})",
                                   sites=np.array([site]))
    if s.flags & _lib.ST_SHIFT:
        raise DomainError("shifted temperature T_bar <= 0")


def _check_region(geom: LatticeGeometry, region):
    """Normalise a (slice_x, slice_y) region in padded coordinates and insist
    it lies inside the physical sites (kernels.py:149-156: ContractViolation
    otherwise)."""
    bounds = []
    for sl, n, phys in ((region[0], geom.NX, geom.phys_x), (region[1], geom.NY, geom.phys_y)):
        lo, hi, step = sl.indices(n)
        if lo < phys.start or hi > phys.stop:
            raise ContractViolation(f"region {region} extends into the halo")
        bounds.append(slice(lo, hi, step))
    return tuple(bounds)


def field_desc(f: PopulationField):
    g = f.geom
    return _lib.field(f.pops, g.Lx, g.Ly, g.Hx, g.Hy)


# ------------------------------------------------------------------ moments --

def moments(f, vs: VelocitySet, check=True):
    """Density, velocity and temperature of a (Q, ...) block (kernels.py:41-71)."""
    t, np_in = _to_device(f)
    torch = _lib.torch_cuda()
    _vs_device(vs, t)
    shape = t.shape[1:]
    b = _block3(t)
    fd = _lib.field(b)
    a, n = b.shape[1], b.shape[2]
    outs = [torch.empty((a, n), dtype=torch.float64, device=t.device) for _ in range(4)]
    st = _status(t.device)
    st.reset()
    _lib.check(_lib.load().tlb_moments(
        fd, _lib.region(0, a, 0, n), *[o.data_ptr() for o in outs], n, int(check),
        st.ptr, _lib.stream_ptr()), "moments")
    rho, ux, uy, T = (o.reshape(shape) for o in outs)
    if check and st.read().flags & _lib.ST_DEGENERATE:
        bad = torch.nonzero(~(rho > 0.0)).cpu().numpy()
        raise DegenerateStateError(f"non-positive density at {bad[:5].tolist()}", sites=bad)
    return tuple(_out(o, np_in) for o in (rho, ux, uy, T))


# -------------------------------------------------------------- equilibrium --

def equilibrium(rho, ux, uy, T, vs: VelocitySet, order=None, check=True):
    """Hermite expansion of the shifted Maxwellian (kernels.py:74-125)."""
    if order is None:
        order = vs.eq_order
    if order not in (2, 3, 4):
        raise DomainError(f"unsupported expansion order {order}")
    torch = _lib.torch_cuda()
    np_in = not any(isinstance(a, torch.Tensor) for a in (rho, ux, uy, T))
    ref = next((a for a in (rho, ux, uy, T) if isinstance(a, torch.Tensor)), None)
    ts = [_to_device(a, ref)[0] for a in (rho, ux, uy, T)]
    ts = torch.broadcast_tensors(*ts)
    shape = ts[0].shape
    flat = [x.reshape(-1).contiguous() for x in ts]
    n = flat[0].numel()
    _vs_device(vs, flat[0])
    out = torch.empty((vs.Q, n), dtype=torch.float64, device=flat[0].device)
    st = _status(flat[0].device)
    st.reset()
    arith = _lib.ARITH["exact"]
    _lib.check(_lib.load().tlb_equilibrium(
        *[x.data_ptr() for x in flat], n, int(order), arith, out.data_ptr(), n,
        int(check), st.ptr, _lib.stream_ptr()), "equilibrium")
    if check:
        _raise_status(st, "equilibrium")
    return _out(out.reshape((vs.Q,) + tuple(shape)), np_in)


# -------------------------------------------------------------- apply_shift --

def apply_shift(ux, uy, T, params: PhysicsParams):
    """Body-force shift u_bar = u + tau g, T_bar = T - tau^2 g^2 / D
    (kernels.py:128-136)."""
    torch = _lib.torch_cuda()
    np_in = not any(isinstance(a, torch.Tensor) for a in (ux, uy, T))
    ref = next((a for a in (ux, uy, T) if isinstance(a, torch.Tensor)), None)
    ts = torch.broadcast_tensors(*[_to_device(a, ref)[0] for a in (ux, uy, T)])
    shape = ts[0].shape
    flat = [x.reshape(-1).contiguous() for x in ts]
    n = flat[0].numel()
    outs = [torch.empty(n, dtype=torch.float64, device=flat[0].device) for _ in range(3)]
    st = _status(flat[0].device)
    st.reset()
    tp = _lib.params(params)
    _lib.check(_lib.load().tlb_apply_shift(
        *[x.data_ptr() for x in flat], n, tp, *[o.data_ptr() for o in outs], st.ptr,
        _lib.stream_ptr()), "apply_shift")
    if st.read().flags & _lib.ST_SHIFT:
        raise DomainError("shifted temperature T_bar <= 0")
    res = [o.reshape(shape) for o in outs]
    if np_in:
        res = [r.cpu().numpy() for r in res]
        if res[0].shape == ():
            res = [float(r) for r in res]
    return tuple(res)


# ------------------------------------------------------------------ collide --

def collide(f, params: PhysicsParams, vs: VelocitySet):
    """BGK relaxation of a gathered (Q, ...) block toward the shifted
    equilibrium (kernels.py:139-146).  Returns a new array."""
    t, np_in = _to_device(f)
    torch = _lib.torch_cuda()
    _vs_device(vs, t)
    b = _block3(t)
    out = torch.empty(b.shape, dtype=torch.float64, device=t.device)
    st = _status(t.device)
    st.reset()
    r = _lib.region(0, b.shape[1], 0, b.shape[2])
    _lib.check(_lib.load().tlb_collide(_lib.field(b), _lib.field(out), r,
                                       _lib.params(params, vs), 0, st.ptr,
                                       _lib.stream_ptr()), "collide")
    _raise_status(st, "collide")
    return _out(out.reshape(t.shape), np_in)


# ---------------------------------------------------------------- propagate --

def propagate(prv: PopulationField, nxt: PopulationField, vs: VelocitySet, region=None):
    """Pull streaming nxt_l(x) = prv_l(x - c_l) on the region
    (kernels.py:168-177).  Mutates nxt in place."""
    geom = prv.geom
    if region is None:
        region = (geom.phys_x, geom.phys_y)
    xs, ys = _check_region(geom, region)
    if xs.stop <= xs.start or ys.stop <= ys.start:
        return
    _vs_device(vs, prv.data)
    _lib.check(_lib.load().tlb_propagate(
        field_desc(prv), field_desc(nxt), _lib.region(xs.start, xs.stop, ys.start, ys.stop),
        _lib.stream_ptr()), "propagate")


# ----------------------------------------------------------------------- bc --

def bc(field: PopulationField, params: PhysicsParams, vs: VelocitySet,
       top=True, bottom=True, x_range=None):
    """Rewrite the 3 rows nearest each wall to the local equilibrium at the
    wall temperature and zero velocity (kernels.py:180-203)."""
    geom = field.geom
    xs = geom.phys_x if x_range is None else x_range
    xs = slice(*xs.indices(geom.NX))
    if not (top or bottom) or xs.stop <= xs.start:
        return
    _vs_device(vs, field.data)
    st = _status(field.device)
    st.reset()
    _lib.check(_lib.load().tlb_bc(field_desc(field), _lib.params(params, vs), int(top),
                                  int(bottom), xs.start, xs.stop, st.ptr,
                                  _lib.stream_ptr()), "bc")
    _raise_status(st, "bc")


# -------------------------------------------------------------------- fused --

def propagate_collide_fused(prv: PopulationField, nxt: PopulationField,
                            params: PhysicsParams, vs: VelocitySet,
                            region=None, exclude_y=()):
    """Gather + collide in one pass; bitwise equal to staged propagate ->
    collide (kernels.py:206-224).  exclude_y lists padded-y [lo, hi) ranges
    the region must not touch."""
    geom = prv.geom
    if region is None:
        region = (geom.phys_x, geom.phys_y)
    xs, ys = _check_region(geom, region)
    for lo, hi in exclude_y:
        if ys.start < hi and ys.stop > lo:
            raise ContractViolation("fused region overlaps bc rows")
    if xs.stop <= xs.start or ys.stop <= ys.start:
        return
    _vs_device(vs, prv.data)
    st = _status(prv.device)
    st.reset()
    _lib.check(_lib.load().tlb_fused(
        field_desc(prv), field_desc(nxt), _lib.region(xs.start, xs.stop, ys.start, ys.stop),
        _lib.params(params, vs), 0, st.ptr, _lib.stream_ptr()), "fused")
    _raise_status(st, "fused")


# --------------------------------------------------------------- monitoring --

def count_negative(f):
    """Number of negative population values (kernels.py:227-229)."""
    t, _ = _to_device(f)
    b = _block3(t)
    st = _status(t.device)
    st.reset()
    _lib.check(_lib.load().tlb_count_negative(
        _lib.field(b), _lib.region(0, b.shape[1], 0, b.shape[2]), st.ptr,
        _lib.stream_ptr()), "count_negative")
    return int(st.read().negatives)
