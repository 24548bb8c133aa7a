"""bench.py's one-JSON-line contract: the reference arm on the CPU (here) and
our arm on the GPU (marked gpu)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def _reference_available():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O

    return O.ref_lib() is not None


@pytest.mark.skipif(not _reference_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("config", ["c1", "c5"])
def test_reference_arm_line(config):
    d = run_bench("--impl", "reference", "--config", config, "--steps", "1", "--warmup", "1")
    assert d["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "dtype", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "reference"
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["unit"] == d["unit"]


@pytest.mark.gpu
def test_our_arm_line_c1():
    d = run_bench("--config", "c1", "--steps", "5", "--warmup", "3", "--no-cpu-baseline")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "gpu_launches", "clocks", "roofline", "e2e"):
        assert k in d, k
    assert d["steps"] == 5 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    assert d["gpu_launches"] > 0 and "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_c5_sweep_line():
    d = run_bench("--config", "c5", "--steps", "1", "--warmup", "1", "--sweep-max", "2200000")
    ops = {(r["op"], tuple(r["grid"])) for r in d["sweep"]}
    assert ("ctransform", (512, 512)) in ops and ("solve_neumann", (128, 128, 128)) in ops
    assert all(r["achieved_gbs"] > 0 and r["ms"] > 0 for r in d["sweep"])
    assert d["unit"] == "GB/s" and d["roofline"]["frac"] > 0
