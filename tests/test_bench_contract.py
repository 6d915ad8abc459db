"""bench.py's JSON line contract, checked on the CPU with the reference arm
(the GPU arm's keys are checked by tests/test_gpu_* runs of bench)."""

import json
import os
import subprocess
import sys

from conftest import ROOT


def test_reference_arm_json_line():
    env = dict(os.environ, OMP_NUM_THREADS="2")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "MLUPS" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]
    with open(os.path.join(ROOT, "BASELINE.json")) as fh:
        assert d["metric"] == json.load(fh)["metric"]


def test_ncu_traffic_reads_the_sidecar_of_a_capture(monkeypatch):
    """bench.ncu_traffic trusts a committed ncu capture only for the SASS hash
    its .sass sidecar records; kernel names contain spaces ("k_tb2<0, 64, 2,
    2, 0> <hash>"), so the hash is the last field."""
    import glob
    import bench
    sidecars = sorted(glob.glob(os.path.join(ROOT, "profiles", "*ncu*_column_raw*.csv.sass")))
    assert sidecars
    with open(sidecars[-1]) as fh:
        name, h = fh.readline().strip().rsplit(" ", 1)
    monkeypatch.setattr(bench, "sass_hash", lambda k: h if k == name else "0" * 16)
    traffic, src = bench.ncu_traffic(name)
    assert traffic is not None and traffic > 0, src
    assert bench.ncu_traffic("k_site<9, 9, 9, 9, 9>")[0] is None
