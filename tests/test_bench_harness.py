"""bench.py's measurement harness on the CPU: the clock sampler reports only
samples inside the timed window (or the nearest ones for windows shorter than
its period) and flags throttle reasons; the reference arm's JSON contract."""
import importlib.util
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def _row(sm, reasons=("Not Active",) * 4):
    return ["0", str(sm), "1965", "500.0", "0x0", *reasons]


def test_sampler_window(bench):
    s = bench.ClockSampler(0)
    s.rows = [(1.0, _row(1000)), (2.0, _row(1965)), (3.0, _row(1965)), (4.0, _row(900))]
    s.window = [1.5, 3.5]
    out = s.summary()
    assert out["sm_mhz"] == 1965.0 and out["samples"] == 2 and out["reasons"] == []


def test_sampler_short_window_uses_neighbours(bench):
    s = bench.ClockSampler(0)
    s.rows = [(1.0, _row(1900)), (2.0, _row(1965))]
    s.window = [1.2, 1.3]
    out = s.summary()
    assert out["samples"] == 2 and out["sm_mhz"] == pytest.approx(1932.5)


def test_sampler_reports_throttle_reasons(bench):
    s = bench.ClockSampler(0)
    s.rows = [(1.0, _row(1500, ("Not Active", "Active", "Not Active", "Active")))]
    s.window = [0.5, 1.5]
    assert s.summary()["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]


def test_sampler_without_samples(bench):
    s = bench.ClockSampler(0)
    s.window = [0.0, 1.0]
    assert s.summary()["sm_mhz"] is None


def test_workloads_named(bench):
    for wl in (bench.WORKLOAD, bench.WORKLOAD_C1, bench.WORKLOAD_C2, bench.WORKLOAD_C3, bench.WORKLOAD_C5):
        assert wl["workload"] and wl["ppb_per_gpu"] > 0 and wl["reduction"] in ("fast", "deterministic")
