"""bench.py's JSON-line contract, on a small workload (C1).

CPU: the reference arm (`--impl reference`, the reference's own engine from
oracle/_ref on the host cores) prints the contract line with `impl`,
`cpu_baseline` and a zero-copy `e2e`.
GPU: our arm prints the full line (roofline, cpu_baseline, e2e, clocks,
gpu_launches) with the B200 engine actually launching kernels.
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _line(args, timeout):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_contract():
    ref = os.path.join(ROOT, "oracle", "_ref", "libsplbref.so")
    if not os.path.exists(ref):
        pytest.skip("oracle/_ref not built")
    d = _line(["--impl", "reference", "--workload", "c1", "--steps", "1", "--warmup", "3"], 300)
    assert BASE_KEYS <= set(d)
    assert d["impl"] == "reference" and d["metric"] == "MSUPS" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "reference" and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "MSUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["warmup"] >= 3


@pytest.mark.gpu
def test_bench_contract():
    d = _line(["--workload", "c1", "--steps", "5", "--warmup", "3", "--no-secondary"], 600)
    assert BASE_KEYS <= set(d)
    assert d["metric"] == "MSUPS" and d["unit"] == "MSUPS" and d["higher_is_better"] is True
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["value"] > 0
    assert d["dtype"] == "f64" and "C1" in d["config"]["workload"]
    roof = d["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s" and roof["peak"] > 0
    assert 0 < roof["frac"] == pytest.approx(roof["achieved"] / roof["peak"])
    cpu = d["cpu_baseline"]
    assert cpu["kind"] == "reference" and cpu["cores"] >= 1 and cpu["value"] > 0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 5  # at least the plain kernel every step
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}


def test_reference_arm_never_maps_the_product():
    """The reference arm times the reference engine alone: its process maps
    oracle/_ref/libsplbref.so and never libsplbcu.so (the C3 sample is
    voxelised by oracle/geometry_gen.py and classified by the reference)."""
    ref = os.path.join(ROOT, "oracle", "_ref", "libsplbref.so")
    if not os.path.exists(ref):
        pytest.skip("oracle/_ref not built")
    code = ("import sys; sys.argv=['bench.py']; import bench; "
            "v = bench.cpu_reference_run('c3', 1, 1.0, 1.0, 1, 'baseline'); "
            "maps = open('/proc/self/maps').read(); "
            "print('REF', 'libsplbref' in maps, 'PRODUCT', 'libsplbcu' in maps, v[3])")
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    line = [x for x in r.stdout.splitlines() if x.startswith("REF")][0].split()
    assert line[1] == "True" and line[3] == "False", line
    assert int(line[4]) == 3478268  # the C3-shaped sample R0=32 L0=160
