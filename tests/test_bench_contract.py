"""bench.py keeps the driver's JSON contract: the reference arm on CPU (here), our arm on a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(args, timeout):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_cpu():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libebl_ref.so")) and \
            not os.path.exists(os.path.join(ROOT, "oracle", "libember_oracle.so")):
        pytest.skip("oracle not built")
    d = _run(["--impl", "reference", "--steps", "1", "--warmup", "1"], 600)
    assert KEYS <= d.keys() and d["impl"] == "reference"
    assert d["metric"] == "cell-updates/sec" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["warmup"] >= 3


@pytest.mark.gpu
def test_our_arm_gpu():
    d = _run(["--steps", "2", "--warmup", "3", "--no-cpu-baseline"], 900)
    assert KEYS <= d.keys() and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == 1024 * 128 * 128
    assert d["gpu_launches"] >= 2 and d["ambiguous_draws"] == 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["config"]["global_batch"] == 1024 and d["config"]["ca_steps"] == 200
