"""bench.py's JSON contract, on CPU: the reference arm end to end on a tiny
row sample (it needs no GPU: the reference simulator in oracle/_ref), and the
committed round-2 bench line (profiles/r02_bench_final.json) against the
keys the driver reads."""
import importlib.util
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench_module():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


BASE_KEYS = ["metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
             "scaling", "vs_baseline", "dtype", "data", "config"]


def test_reference_arm_line():
    if not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libref_sim.so")):
        pytest.skip("oracle/_ref not built (needs /root/reference)")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-stride", "4096"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in BASE_KEYS:
        assert k in line, k
    assert line["unit"] == "GTEPS" and line["higher_is_better"] is True and line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"] and cb["sample"]
    assert line["e2e"] == {"value": line["value"], "unit": "GTEPS", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert "no product library" in line["config"]["input"]


def test_committed_bench_line_keys():
    with open(os.path.join(ROOT, "profiles", "r02_bench_final.json")) as f:
        line = json.load(f)
    for k in BASE_KEYS + ["roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"]:
        assert k in line, k
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and roof["unit"] == "GB/s"
    assert roof["frac"] == pytest.approx(roof["achieved"] / roof["peak"], rel=1e-3)
    # achieved = algorithmic bytes / step time
    assert roof["achieved"] == pytest.approx(roof["algorithmic_bytes"] / (line["ms_per_step"] * 1e-3) / 1e9,
                                             rel=0.01)
    assert roof["traffic"] and 0.9 < roof["traffic"] / roof["algorithmic_bytes"] < 1.1
    assert line["cpu_baseline"]["kind"] in ("port", "reference") and line["cpu_baseline"]["cores"] >= 1
    e2e = line["e2e"]
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0 and e2e["value"] > 0
    assert line["gpu_launches"] > 0
    assert set(line["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    assert line["parity"]["grid_vs_fp64_rtol_1e-5"] is True and "parity_failed" not in line
    # GTEPS = nnz / time
    assert line["value"] == pytest.approx(line["config"]["nnz"] / (line["ms_per_step"] * 1e-3) / 1e9, rel=0.01)


def test_summary_of_committed_line():
    with open(os.path.join(ROOT, "profiles", "r02_bench_final.json")) as f:
        line = json.load(f)
    s = _bench_module()._summary(line)
    assert s["spmv_gteps"] == line["value"] and s["roofline_frac"] == line["roofline"]["frac"]
    assert s["apps"]["sssp"]["vs_basic"] == line["apps"]["sssp"]["best_vs_basic"]
    assert s["parity_failed"] == []
