"""Host-side pieces of bench.py (no GPU): workload scaling rules, the exchange
summary, and the measured-traffic scaling from profiles/traffic.json."""

import json
import os

import pytest

import bench

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,world,dp,sp,gbs", [
    ("cfg2", 1, 1, 1, 4), ("cfg2", 4, 4, 1, 16), ("cfg2", 8, 8, 1, 32),
    ("cfg4", 8, 2, 4, 16), ("cfg4", 2, 2, 1, 16), ("cfg5", 4, 4, 1, 8)])
def test_weak_scaling_workload(name, world, dp, sp, gbs):
    cfg, d, s, g = bench.workload(name, world)
    assert (d, s, g) == (dp, sp, gbs)
    assert d * s == world


def test_exchange_summary():
    info = [dict(disp_bytes=100, disp_remote=25, ret_bytes=1000, ret_remote=100),
            dict(disp_bytes=300, disp_remote=75, ret_bytes=3000, ret_remote=900)]
    x = bench.exchange_summary(info, [0, 1, 1], rank=2)
    assert x["rank"] == 2
    assert x["dispatch_bytes"] == pytest.approx(700 / 3)
    assert x["dispatch_remote_frac"] == pytest.approx(0.25)
    assert x["return_remote_frac"] == pytest.approx(1900 / 7000)


def test_captured_traffic_reports_the_capture():
    rec = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    for name in ("cfg2", "target1"):
        r = rec[name]
        t, src = bench.captured_traffic(name)
        assert t == r["dram_read"] + r["dram_write"] and "ncu" in src
        assert 0.5 < t / r["algorithmic_bytes"] < 1.2  # no wasted re-reads
    t, src = bench.captured_traffic("no_such_config")
    assert t is None and "no ncu capture" in src


def test_tensor_peak_follows_the_clock_record():
    _, burst, sus, _ = bench.peaks()
    full = {"sm_mhz": 1965.0, "sm_max_mhz": 1965.0, "reasons": []}
    assert bench.choose_tensor_peak(full)[0] == burst
    capped = dict(full, reasons=["sw_power_cap"])
    assert bench.choose_tensor_peak(capped)[0] == sus
    slow = dict(full, sm_mhz=1300.0)
    assert bench.choose_tensor_peak(slow)[0] == sus


def test_both_arms_print_the_same_config():
    """The reference arm and ours time the same distinct steps in the same order
    and print the same `config` dict (the driver compares them)."""
    class A:
        steps, warmup, distinct = 20, 5, 8
    n = bench.n_distinct_of(A)
    assert n == 8 and bench.timed_indices(A, n)[:4] == [5, 6, 7, 0]
    a = bench.config_dict("cfg2", 1, n, 43355.0, 55499.25)
    b = bench.config_dict("cfg2", 1, n, 43355.0, 55499.25)
    assert a == b and a["workload"] == "cfg2" and a["global_batch"] == 4


def test_balance_summary():
    import numpy as np
    info = [dict(pre=np.array([10.0, 2.0]), post=np.array([6.0, 6.0])),
            dict(pre=np.array([4.0, 4.0]), post=np.array([5.0, 3.0]))]
    b = bench.balance_summary(info, [0, 1])
    assert b["pre_loads_first_step"] == [10.0, 2.0]
    assert b["pre_imbalance"] == pytest.approx((10 / 6 + 1) / 2)
    assert b["post_imbalance"] == pytest.approx((1 + 5 / 4) / 2)


def test_combined_bound_per_step():
    """The exchange roofline: per step the slower of HBM and NVLink on the
    slowest rank, then the mean over steps (an NVLink-bound step is not hidden
    by averaging the byte matrices first)."""
    import numpy as np
    MB = 1e6
    # step 0: rank 1 pushes 70 MB to rank 0 (NVLink-bound); step 1: all local
    s0 = np.array([[100 * MB, 0], [70 * MB, 60 * MB]])
    s1 = np.array([[200 * MB, 0], [0, 200 * MB]])
    r = bench.combined_bound([s0, s1], hbm_gbs=6500.0, link_gbs=700.0, t_ms=0.2)
    b0 = max(70 * MB / 700e9, (2 * 100 * MB + 70 * MB) / 6500e9) * 1e3  # rank 0: ingress
    b0 = max(b0, (2 * 60 * MB + 70 * MB) / 6500e9 * 1e3)
    b1 = 2 * 200 * MB / 6500e9 * 1e3
    assert r["bound_ms_per_step"] == pytest.approx([b0, b1])
    assert r["bound_ms"] == pytest.approx((b0 + b1) / 2)
    assert r["frac"] == pytest.approx((b0 + b1) / 2 / 0.2)
    assert r["steps_nvlink_bound"] == 1
    avg = bench.combined_bound([(s0 + s1) / 2], 6500.0, 700.0, 0.2)["bound_ms"]
    assert avg < r["bound_ms"]  # averaging first understates the bound
