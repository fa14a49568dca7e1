"""The bench JSON line keeps the driver's contract (CPU): the last line
recorded on a B200 (profiles/r02q_bench_c2.json) carries every key the
contract names, with consistent values."""

import json
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LINE = os.path.join(ROOT, "profiles", "r02q_bench_c2.json")


@pytest.fixture(scope="module")
def line():
    if not os.path.exists(LINE):
        pytest.skip("no recorded bench line")
    return json.loads(open(LINE).read())


def test_top_level_keys(line):
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert k in line, k
    assert line["higher_is_better"] is True and line["scaling"] in ("weak", "strong")
    assert line["warmup"] >= 3 and line["n_gpus"] >= 1
    assert abs(line["ms_per_step"] - 1e3 / line["value"] * line["n_gpus"]) < 1e-6 * 1e3


def test_config_names_the_workload(line):
    cfg = line["config"]
    assert cfg["workload"].startswith("C2:")
    assert "l2" in cfg and cfg["inputs_match_reference_digest"] is True


def test_roofline_block(line):
    r = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert r["bound"] in ("hbm", "tensor") and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9


def test_cpu_baseline_and_e2e(line):
    c = line["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] in ("reference", "port")
    e = line["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["value"] != line["value"]  # measured separately, through host buffers


def test_clocks_and_launches(line):
    cl = line["clocks"]
    for k in ("sm_mhz", "sm_max_mhz", "reasons"):
        assert k in cl, k
    assert not set(cl["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    assert line["gpu_launches"] > 0
