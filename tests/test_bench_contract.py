"""The bench.py JSON-line contract (the driver parses it): the reference arm on CPU, the GPU arm on a
B200 (small cfg1 instance so the test runs in seconds)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


BASE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config")


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--config", "cfg1", "--steps", "1", "--warmup", "1")
    for key in BASE_KEYS:
        assert key in d, key
    assert d["impl"] == "reference" and d["config"]["workload"] == "cfg1"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1


@pytest.mark.gpu
def test_gpu_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = run_bench("--config", "cfg1", "--steps", "3", "--warmup", "3", "--no-cpu-baseline")
    for key in BASE_KEYS:
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3
    assert d["config"]["workload"] == "cfg1" and d["dtype"] == "f32"
    r = d["roofline"]
    for key in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert key in r, key
    assert 0.0 < r["frac"] and r["achieved"] > 0
    assert set(r["per_kernel"]) >= {"k_forward", "k_adjoint_mp"}
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] == 4
    assert d["gpu_launches"] == 7 * 3  # gather, forward, reduce, loss, moment prep, adjoint, gather + update
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
