"""bench.py contract: helpers on CPU; on the GPU a tiny run of both arms, one
rank and two ranks under torchrun (ranks share the device over gloo)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def test_algorithmic_bytes_formula():
    import bench
    from paper_2604_16402_b200 import _lib as L
    st = np.zeros(2, dtype=L.STATS_DTYPE)
    st["dist_evals"] = [10, 20]
    st["expanded"] = [4, 8]
    st["gathered"] = [100, 0]
    st["seed_attempts"] = [128, 128]
    got = bench.algorithmic_bytes(st, dp=128, k_max=32, k=10)
    want = 4 * 128 * 30 + 4 * 32 * 12 + 8 * 100 + 8 * 256 + 2 * (4 * 128 + 16 * 10)
    assert got == want


def test_clock_summary_flags_throttle_reasons():
    import bench
    c = bench.ClockSampler.__new__(bench.ClockSampler)
    c._nv = None
    c.rows = [(1965.0, 1965.0, 0x0), (1800.0, 1965.0, 0x4), (1900.0, 1965.0, 0x40)]
    s = c.summary()
    assert s["sm_max_mhz"] == 1965.0 and s["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]


SMALL = ["--rows", "20000", "--nq", "500", "--cap", "2000", "--steps", "3", "--warmup", "3", "--insert-batch", "2000"]


def _line(out: str) -> dict:
    return json.loads([x for x in out.splitlines() if x.startswith("{")][-1])


@pytest.mark.gpu
def test_bench_single_rank_line():
    r = subprocess.run([sys.executable, "bench.py", *SMALL, "--cpu-sample", "32"], capture_output=True, text=True,
                       cwd=ROOT, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "dtype", "config", "e2e", "roofline", "cpu_baseline", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["steps"] == 3 and d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 6
    assert d["roofline"]["unit"] == "GB/s" and 0 < d["roofline"]["frac"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    # the CPU baseline (the reference's algorithm) returns the GPU's results exactly
    assert d["cpu_baseline"]["result_agreement"] == 1.0


@pytest.mark.gpu
def test_bench_two_ranks_and_reference_arm_under_torchrun():
    env = dict(os.environ, GRAB_BENCH_SHARED_GPU="1")
    base = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
            "127.0.0.1"]
    r = subprocess.run(base + ["--master-port", "29621", "bench.py", "--gpus", "2", *SMALL, "--no-cpu"],
                       capture_output=True, text=True, cwd=ROOT, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0
    r = subprocess.run(base + ["--master-port", "29622", "bench.py", "--impl", "reference", "--gpus", "2", *SMALL],
                       capture_output=True, text=True, cwd=ROOT, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "port" and d["steps"] == 3
