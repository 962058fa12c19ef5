"""bench.py keeps the driver's JSON-line contract: the reference arm on CPU, our arm on
the GPU (short kernels-only run).  Guards the key set, not the numbers."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "0")
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["config"]["workload"] == "resnet50-lasgd-sync" and d["value"] > 0 and d["higher_is_better"] is True
    cb = d["cpu_baseline"]
    assert {"value", "unit", "cores", "kind", "sample"} <= set(cb) and cb["kind"] in ("port", "reference")
    assert cb["value"] == d["value"] and cb["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_our_arm_line():
    d = _run("--steps", "5", "--warmup", "3", "--kernels-only", "--no-cpu-baseline")
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["scaling"] == "weak"
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and r["bound"] in ("hbm", "nvlink")
    assert 0 < r["frac"] <= 1.05 and r["unit"] == "GB/s"
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["h2d_bytes_per_step"] == 4 * d["config"]["params"] and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] == 5  # one fused round per step at N = 1
    assert d["clocks"] is None or {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_reference_arm_records_our_config():
    """Both arms name the same config (the driver compares them): the reference arm's
    fused_round_algo is what our arm's communicator resolves at that world size."""
    sys.path.insert(0, ROOT)
    import bench

    assert bench.fused_algo_name(1, 25_557_032) == "oneshot"
    assert bench.fused_algo_name(2, 25_557_032) == "push"
    assert bench.fused_algo_name(2, 3_504_872) == "oneshot"
    assert bench.fused_algo_name(4, 25_557_032) == "push"
    assert bench.fused_algo_name(4, 1_000_000) == "oneshot"
    assert bench.fused_algo_name(8, 3_504_872) == "push"


def test_fused_algo_name_matches_the_communicator():
    sys.path.insert(0, ROOT)
    import bench
    from paper_2203_13085_b200 import _native as N

    for P in range(2, 9):
        for n in (262_144, 2_097_152, 3_504_872, 11_181_642, 25_557_032):
            got = N.lib().lasgd_resolve_fused_algo_for(P, 4 * n)
            assert {1: "oneshot", 2: "twoshot", 3: "push"}[got] == bench.fused_algo_name(P, n), (P, n)


def test_exposed_stats_pairs_blocks_and_ignores_level_switches():
    """The training legs' exposed-sync estimator: median of paired per-repetition
    differences; a level switch of the whole step (both legs shift together) cancels,
    one switch between the two blocks of a repetition is an outlier the median ignores."""
    sys.path.insert(0, ROOT)
    import bench

    base = [51.30] * 12 + [51.70] * 12
    leg = [b + 0.08 for b in base]
    leg[5] += 0.40  # the switch fell between the two blocks of repetition 5
    d = bench._exposed_stats(leg, base)
    assert abs(d["median"] - 0.08) < 1e-9
    assert d["ci95"][0] - 1e-9 <= 0.08 <= d["ci95"][1] + 1e-9 and d["ci95_halfwidth"] < 0.01
    assert d["blocks"] == 24
