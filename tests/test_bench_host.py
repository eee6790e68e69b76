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


def test_measured_traffic_scales_the_captured_ratio():
    rec = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    for name in ("cfg2", "target1"):
        r = rec[name]
        ratio = (r["dram_read"] + r["dram_write"]) / r["algorithmic_bytes"]
        assert 0.5 < ratio < 1.2  # reads equal the algorithmic bytes; writes partly in L2
        t, src = bench.measured_traffic(name, 1e9)
        assert t == pytest.approx(1e9 * ratio) and "ncu" in src
    t, src = bench.measured_traffic("no_such_config", 1e9)
    assert t is None and "no ncu capture" in src
