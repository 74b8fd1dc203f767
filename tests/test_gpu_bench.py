"""bench.py's own arm on the GPU (config 3, so it runs in seconds): one JSON line with the
contract's keys, a positive value, the roofline / clocks / launch-count objects, and e2e +
solve blocks when enabled."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*extra):
    r = subprocess.run([sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--no-cpu",
                        *extra], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return lines[0]


def test_bench_line_contract_small():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    j = _run("--workload", "c3_poisson5d", "--e2e-steps", "1", "--e2e-ring-rows", "8192",
             "--per-config-budget", "3")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "gpu_launches", "clocks", "e2e", "solve"):
        assert k in j, k
    assert j["value"] > 0 and j["n_gpus"] == 1 and j["steps"] == 3 and j["warmup"] == 3
    rf = j["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert 0 < rf["frac"] < 1.5 and rf["bound"] == "hbm"
    assert j["gpu_launches"] >= 2 * j["steps"]
    assert j["e2e"]["value"] > 0 and j["e2e"]["d2h_bytes_per_step"] > 0
    assert j["solve"]["ms"] > 0
    assert "sm_mhz" in j["clocks"] and "reasons" in j["clocks"]
    assert j["e2e_device_resident"]["value"] > 0 and j["e2e_device_resident"]["h2d_bytes_per_step"] > 0
    pc = j["per_config"]                       # bounded: later configs may be skipped
    assert set(pc) == {"c1_poisson1d", "c2_poisson2d", "c3_poisson5d", "c4_heat2d", "c5_biharm3d"}
    c1 = pc["c1_poisson1d"]
    assert c1["graph_us_per_step"] > 0 and 0 < c1["frac_of_copy_peak"] < 1.5
    assert c1["solve_ms"]["ms"] > 0 and c1["rel_l2_vs_u_star"] < 1e-6
    assert all(("skipped" in v) or v["graph_us_per_step"] > 0 for v in pc.values())


def test_cli_solves_a_config():
    """python -m paper_2602_10541_b200 <config>: Algorithm 1 end to end, u* recovered"""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, "-m", "paper_2602_10541_b200", "c1_poisson1d"], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout)
    assert out["rows"] == 1002 and out["features"] == 500
    assert out["rel_l2_vs_u_star"] < 1e-6 and out["solve_ms"] > 0
