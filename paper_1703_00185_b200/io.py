"""Snapshot writers, tables and YAML configs (reference io.py:13-80).

The observables come off the device already reduced: ``write_pgm`` of a
device field runs the min/max + 8-bit quantisation on the GPU
(``tlb_pgm_image``) and copies only the image bytes; numpy inputs take the
same kernel after an upload.  Byte-identical to the reference's image
(numpy's round-half-even == rint).
"""

import csv

import numpy as np

from . import _lib
from .errors import ConfigurationError
from .geometry import MacroFields


def pgm_bytes(values):
    """The P5 image of a (Lx, Ly) field as bytes (header + pixels)."""
    torch = _lib.torch_cuda()
    t = values if isinstance(values, torch.Tensor) else torch.as_tensor(
        np.ascontiguousarray(values, dtype=np.float64), device="cuda")
    t = t.to(torch.float64)
    if t.dim() != 2 or t.stride(1) != 1:
        t = t.reshape(t.shape[0], -1).contiguous()
    nx, ny = t.shape
    mm = torch.empty(2, dtype=torch.int64, device=t.device)
    img = torch.empty(nx * ny, dtype=torch.uint8, device=t.device)
    _lib.check(_lib.load().tlb_pgm_image(t.data_ptr(), nx, ny, t.stride(0), mm.data_ptr(),
                                         img.data_ptr(), _lib.stream_ptr()), "pgm image")
    return f"P5\n{nx} {ny}\n255\n".encode() + bytes(img.cpu().numpy())


def write_pgm(path, values):
    """P5 snapshot of a (Lx, Ly) field: min-max scaled to 0..255, first
    image row = largest y (reference io.py:13-24, same bytes)."""
    with open(path, "wb") as fh:
        fh.write(pgm_bytes(values))


def _host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


_MACRO_HEADER = ("x [site]", "y [site]", "rho [lattice]", "ux [lattice]",
                 "uy [lattice]", "T [lattice]")
_METRIC_HEADER = ("step", "rank", "t_comm_nc [s]", "t_comm_c [s]", "t_bulk [s]",
                  "t_border [s]", "negative_populations [count]")


def _csv(path, header, rows):
    with open(path, "w", newline="") as fh:
        out = csv.writer(fh)
        out.writerow(list(header))
        out.writerows(rows)


def write_macro_csv(path, macro: MacroFields):
    """One CSV row per site, x-major, values as Python float reprs (the
    reference's format, io.py:27-40); device fields are copied back once."""
    cols = [_host(getattr(macro, k)) for k in ("rho", "ux", "uy", "T")]
    nx, ny = cols[0].shape

    def rows():
        for x in range(nx):
            for y in range(ny):
                yield [x, y] + [repr(float(c[x, y])) for c in cols]

    _csv(path, _MACRO_HEADER, rows())


def write_table(path, header, rows):
    """Plain CSV: a header row then the rows (reference io.py:43-47)."""
    _csv(path, header, rows)


def write_metrics(path, metrics):
    """Per-(step, rank) metrics table in the reference CLI's format
    (cli.py:69-75)."""
    times = ("t_comm_nc", "t_comm_c", "t_bulk", "t_border")
    _csv(path, _METRIC_HEADER,
         ([m["step"], m["rank"]] + [repr(m[k]) for k in times] + [m["negatives"]]
          for m in metrics))


def load_config(path):
    """A YAML mapping of run settings (reference io.py:72-80)."""
    import yaml
    try:
        with open(path) as fh:
            cfg = yaml.safe_load(fh)
    except FileNotFoundError:
        raise ConfigurationError(f"config file {path!r} not found") from None
    if isinstance(cfg, dict):
        return cfg
    raise ConfigurationError(f"{path}: expected a key/value mapping")
