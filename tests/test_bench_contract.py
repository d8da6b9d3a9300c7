"""bench.py keeps the driver's JSON contract: the reference arm on CPU (here), our arm on a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}

# runs bench.py's main in-process, then reports which shared objects the process mapped
_WRAP = """
import runpy, sys, json
sys.argv = ["bench.py"] + sys.argv[1:]
try:
    runpy.run_path("bench.py", run_name="__main__")
except SystemExit as e:
    assert not e.code, e.code
maps = open("/proc/self/maps").read()
print("MAPS " + json.dumps(sorted({l.split()[-1] for l in maps.splitlines() if l.endswith(".so")})))
"""


def _run(args, timeout):
    out = subprocess.run([sys.executable, "-c", _WRAP] + args, capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    maps = json.loads([l for l in out.stdout.splitlines() if l.startswith("MAPS ")][0][5:])
    return json.loads(lines[0]), maps


def _ref_built():
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libebl_ref.so"))


@pytest.mark.parametrize("config", ["C1", "C2", "C4"])
def test_reference_arm_cpu(config):
    """The reference arm runs the reference's own code (oracle/_ref) with inputs from the oracle's
    generator: the product library is never loaded, and the config block equals our arm's."""
    if not _ref_built():
        pytest.skip("reference not built here (oracle/_ref)")
    d, maps = _run(["--impl", "reference", "--config", config, "--steps", "1", "--warmup", "1"], 900)
    assert KEYS <= d.keys() and d["impl"] == "reference"
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["warmup"] >= 3
    assert not [m for m in maps if "ember_b200" in m or "emberline_b200" in m], maps
    assert any("libebl_ref.so" in m for m in maps)
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.config_json(config, 1, "weak")
    assert d["metric"] == bench.SPEC[config]["metric"]


def test_config_blocks_identical_across_arms():
    sys.path.insert(0, ROOT)
    import bench
    for c in bench.SPEC:
        for world in (1, 2, 8):
            for sc in ("weak", "strong"):
                a = bench.config_json(c, world, sc)
                assert "kernel" not in a and a == bench.config_json(c, world, sc)
    assert bench.config_json("C1", 8, "strong")["envs_per_rank"] == 128
    assert bench.config_json("C1", 8, "weak")["global_batch"] == 8192
    # strong scaling: the rank ranges tile the batch exactly
    for world in (1, 2, 3, 8):
        got = [bench.rank_envs("C1", r, world, "strong") for r in range(world)]
        assert sum(n for _, n in got) == 1024 and got[0][0] == 0
        assert all(got[i][0] + got[i][1] == got[i + 1][0] for i in range(world - 1))


@pytest.mark.gpu
def test_our_arm_gpu():
    d, maps = _run(["--steps", "2", "--warmup", "3", "--no-cpu-baseline"], 900)
    assert KEYS <= d.keys() and d["impl"] == "ours"
    assert d["n_gpus"] == 1 and d["steps"] == 2 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "issue" and r["kernel"] == "k_step_warp" and r["hbm"]["alg_frac"] > 0
    if r["achieved"] is not None:
        assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == 1024 * 128 * 128
    assert d["gpu_launches"] >= 2 and d["ambiguous_draws"] == 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"]
    assert d["config"]["global_batch"] == 1024 and d["config"]["steps_per_run"] == 200
    assert any("libember_b200.so" in m for m in maps)


@pytest.mark.gpu
@pytest.mark.parametrize("config", ["C0", "C2", "C3", "C4"])
def test_our_arm_gpu_side_configs(config):
    d, _ = _run(["--config", config, "--steps", "2", "--warmup", "3", "--no-cpu-baseline"], 900)
    assert KEYS <= d.keys() and d["value"] > 0 and d["gpu_launches"] >= 1
    r = d["roofline"]
    # shared-memory-resident kernels (C2 rollout, C3 tiles) are bound by issue, not by HBM
    assert r["bound"] == ("issue" if config in ("C2", "C3") else "hbm")
    assert r["frac"] is None or 0 < r["frac"] <= 1.0, r
    if config == "C3":
        assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == 16384 * 16384
