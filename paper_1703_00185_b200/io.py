"""Snapshot output and config loading (io.py of the reference, io.py:13-80).

The observables come off the device already reduced: ``write_pgm`` of a
device field runs the min/max + 8-bit quantisation on the GPU
(``tlb_pgm_image``) and copies only the image bytes; numpy inputs take the
same kernel after an upload.  Byte-identical to the reference's image
(numpy's round-half-even == rint).
"""

import csv
import os

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
    """8-bit binary PGM (P5) of a (Lx, Ly) scalar field, min-max normalised;
    image rows run top to bottom (decreasing lattice y) (io.py:13-24)."""
    data = pgm_bytes(values)
    with open(path, "wb") as fh:
        fh.write(data)


def _host(a):
    return a.cpu().numpy() if hasattr(a, "cpu") else np.asarray(a)


def write_macro_csv(path, macro: MacroFields):
    """Row-major CSV of the macroscopic fields with a labelled header
    (io.py:27-40)."""
    rho, ux, uy, T = (_host(a) for a in (macro.rho, macro.ux, macro.uy, macro.T))
    Lx, Ly = rho.shape
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["x [site]", "y [site]", "rho [lattice]", "ux [lattice]",
                    "uy [lattice]", "T [lattice]"])
        for x in range(Lx):
            for y in range(Ly):
                w.writerow([x, y, repr(float(rho[x, y])), repr(float(ux[x, y])),
                            repr(float(uy[x, y])), repr(float(T[x, y]))])


def write_table(path, header, rows):
    """io.py:43-47."""
    with open(path, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(header)
        w.writerows(rows)


def write_metrics(path, metrics):
    """Per-(step, rank) metrics table in the reference CLI's format
    (cli.py:69-75)."""
    write_table(path, ["step", "rank", "t_comm_nc [s]", "t_comm_c [s]", "t_bulk [s]",
                       "t_border [s]", "negative_populations [count]"],
                [[m["step"], m["rank"], repr(m["t_comm_nc"]), repr(m["t_comm_c"]),
                  repr(m["t_bulk"]), repr(m["t_border"]), m["negatives"]] for m in metrics])


def load_config(path):
    """YAML run configuration: a mapping of explicit keys (io.py:72-80)."""
    import yaml
    if not os.path.exists(path):
        raise ConfigurationError(f"config file {path!r} not found")
    with open(path) as fh:
        data = yaml.safe_load(fh)
    if not isinstance(data, dict):
        raise ConfigurationError(f"{path}: expected a key/value mapping")
    return data
