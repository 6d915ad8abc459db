"""The exact arithmetic replaces IEEE divisions by Markstein-corrected
reciprocal products (csrc/d2q37.cuh).  This checks the identities on the CPU
(same IEEE binary64 fma semantics) over 6e7 random operands; the GPU parity
tests then check the kernels bit for bit."""

import os
import subprocess

from conftest import ROOT


def test_markstein_division_identities(tmp_path):
    exe = tmp_path / "markstein"
    subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-o", str(exe),
                    os.path.join(ROOT, "tests", "c", "markstein.c"), "-lm"], check=True)
    out = subprocess.run([str(exe), "10000000"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert out.stdout.startswith("0 mismatches")
