"""The bench JSON contract, checked on the committed B200 results (no GPU).

bench.py prints one JSON line that the round driver parses; this pins its keys,
units and internal consistency on `results/r2_bench.json` (the last measured
line of round 2) so a refactor of bench.py cannot silently drop a field.
"""
import json
import os

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def _line(name):
    path = os.path.join(ROOT, "results", name)
    if not os.path.exists(path):
        pytest.skip(f"{name} not committed")
    with open(path) as fh:
        return json.loads(fh.read().strip().splitlines()[-1])


def test_bench_line_keys_and_consistency():
    d = _line("r2_bench.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["unit"] == "GRays/s" and d["higher_is_better"] is True and d["warmup"] >= 3
    assert d["config"]["workload"].startswith("config3_pair")
    n, m, dd = d["config"]["n"], d["config"]["n_angles"], d["config"]["n_detectors"]
    # value = rays per step / step time
    assert abs(m * dd / (d["ms_per_step"] * 1e-3) / 1e9 - d["value"]) <= 1e-6 * d["value"]
    e = d["e2e"]
    assert e["unit"] == d["unit"] and e["h2d_bytes_per_step"] == 4 * (n * n + m * dd)
    assert e["verified_against_device"] is True
    # the drop-in call (numpy in / out through w @ x, w.T @ y) is the headline e2e;
    # the pipelined pinned-buffer schedule is reported beside it
    assert "w @ x" in e["call"] and d["e2e_pipelined"]["verified_against_device"] is True
    r = d["roofline"]
    assert r["bound"] == "gather" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    # exact nnz per launch over the dominant kernel's time
    t_dom = max(d["kernels_ms"].values()) * 1e-3
    assert abs(r["updates_per_launch"] / t_dom / 1e9 - r["achieved"]) <= 1e-3 * r["achieved"]
    assert r["peak"] == pytest.approx(r["n_sm"] * 32 * r["f_sm_mhz"] * 1e-3)
    # formula (4/pi) m n^2 within 1e-5 of the exact count
    nz = d["nnz"]
    assert abs(nz["formula_local"] - nz["exact_local"]) <= 1e-5 * nz["exact_local"]
    # value: the dependent (one-stream) pair a Krylov iteration uses; the two
    # independent products on two streams are reported beside it
    assert d["value"] == d["value_sequential"] and "dependent" in d["pair_schedule"]
    assert abs(m * dd / (d["ms_per_step_two_streams"] * 1e-3) / 1e9 - d["value_two_streams"]) \
        <= 1e-6 * d["value_two_streams"]
    assert "host" in d["cpu_baseline"] and d["cpu_baseline"]["host"]["cpu_model"]
    cb = d["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["sample"]
    assert d["gpu_launches"] > 0
    assert not set(d["clocks"]["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown",
                                              "sw_thermal_slowdown"}
    w = d["wmg_cgls"]
    assert w["status"] == "converged" and w["final_rel_residual"] < 1e-4


def test_reference_arm_line():
    d = _line("r2_bench_reference.json")
    assert d["impl"] == "reference" and d["unit"] == "GRays/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["cpu_baseline"]["value"] == d["value"]
