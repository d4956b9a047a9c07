"""bench.py's output contract (the driver parses it): the JSON line's keys and
their consistency, for the CPU reference arm (here) and the GPU arm (-m gpu,
single GPU and two loopback ranks)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_bench(*args, timeout=900):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [x for x in out.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]  # ONE JSON line
    return json.loads(lines[0])


BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def check_common(d, steps, warmup, n_gpus):
    assert BASE_KEYS <= set(d), BASE_KEYS - set(d)
    assert d["unit"] == "steps/s" and d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == steps and d["warmup"] == warmup and d["n_gpus"] == n_gpus
    assert d["dtype"] == "f64" and d["data"] == "synthetic" and d["scaling"] in ("weak", "strong")
    assert d["config"]["workload"] == "sparse5000x3000_k10"
    assert d["ms_per_step"] > 0
    e = d["e2e"]
    if e is not None or "comm" not in d:  # (the loopback harness line has no e2e)
        assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e) and e["unit"] == d["unit"]


def test_reference_arm_line():
    d = run_bench("--impl", "reference", "--workload", "1", "--steps", "1", "--warmup", "0", timeout=600)
    check_common(d, 1, 0, 1)
    assert d["impl"] == "reference"
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"] and cb["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"]
    assert {"workload", "m", "n", "nnz", "k", "t", "tol", "maxit", "l2", "parallelism", "reorth"} == set(d["config"])


@pytest.mark.gpu
def test_gpu_arm_line():
    d = run_bench("--workload", "1", "--steps", "2", "--warmup", "3")
    check_common(d, 2, 3, 1)
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r)
    assert r["bound"] in ("hbm", "tensor", "alu") and r["unit"] in ("GB/s", "TFLOP/s")
    assert abs(r["frac"] - r["achieved"] / r["peak"]) <= 1e-9 * max(1.0, r["frac"])
    assert d["gpu_launches"] > 0
    c = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(c)
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["value"] > 0
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0
    assert d["run"]["lanczos_steps_per_solve"] > 0 and d["run"]["time_to_k_ms"] > 0
    # `config` names the workload only: the reference arm prints the same dict
    ref = run_bench("--impl", "reference", "--workload", "1", "--steps", "1", "--warmup", "0", timeout=600)
    assert ref["config"] == d["config"]


@pytest.mark.gpu
def test_gpu_arm_two_loopback_ranks():
    d = run_bench("--gpus", "2", "--comm", "loopback", "--workload", "1", "--steps", "1", "--warmup", "3", "--no-cpu")
    check_common(d, 1, 3, 2)


@pytest.mark.gpu
def test_gpu_arm_rows_e2e():
    """The multi-GPU e2e leg (rows of A in, U/S/V rows out around svdsc_matrix_csr +
    svdsc_solve; the default for --gpus > 1) on one GPU."""
    d = run_bench("--workload", "1", "--steps", "1", "--warmup", "3", "--no-cpu", "--e2e-rows")
    check_common(d, 1, 3, 1)
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 12 * 150000 and e["d2h_bytes_per_step"] > 8 * 10 * 8000

