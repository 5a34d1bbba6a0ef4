"""The reference's compute_metrics known answers (pkg/tests/test_engine.py:240-283)
against the host-side mirror compute_metrics (the definition the device
co_metrics path is pinned to in tests/test_metrics_device.py)."""
import pytest

from paper_2503_13773_b200 import Lifecycle, Request, RequestRuntime, compute_metrics

BIG_SLO = 10**9


def mk_req(rid=0, arrival=0, prompt=10, out=3, ttft=BIG_SLO, tbt=BIG_SLO):
    return Request(id=rid, arrival_us=arrival, prompt_len=prompt, true_output_len=out,
                   slo_ttft_us=ttft, slo_tbt_us=tbt)


def _manual_runtime(times_us, arrival=0):
    rt = RequestRuntime()
    rt.token_times_us = list(times_us)
    rt.first_token_at_us = times_us[0]
    rt.last_token_at_us = times_us[-1]
    rt.first_start_us = arrival
    rt.completion_us = times_us[-1]
    return rt


def test_compute_metrics_closed_form():
    # test_engine.py:250-268
    good = mk_req(rid=0, prompt=5, out=3, ttft=15_000, tbt=15_000)
    good.state = Lifecycle.COMPLETED
    bad = mk_req(rid=1, prompt=5, out=3, ttft=15_000, tbt=15_000)
    runtimes = {0: _manual_runtime([10_000, 20_000, 30_000]), 1: RequestRuntime()}
    report = compute_metrics(requests={0: good, 1: bad}, runtimes=runtimes, policy="cacheopt", seed=0,
                             makespan_us=30_000, capacity_tokens=1024, samples=[(100, 80)])
    assert report.completed == 1
    assert report.ttft_us["p50"] == 10_000
    assert report.tbt_us["p50"] == 10_000 and report.tbt_us["max"] == 10_000
    assert report.ttft_attainment == 0.5
    assert report.tbt_attainment == 0.5
    assert report.normalized_us_per_token["mean"] == pytest.approx(10_000)
    assert report.kvc_utilization_mean == pytest.approx(100 / 1024)


def test_compute_metrics_flags_tbt_violation():
    # test_engine.py:271-283
    req = mk_req(rid=0, prompt=5, out=3, ttft=15_000, tbt=9_000)
    req.state = Lifecycle.COMPLETED
    report = compute_metrics(requests={0: req}, runtimes={0: _manual_runtime([10_000, 20_000, 30_000])},
                             policy="cacheopt", seed=0, makespan_us=30_000, capacity_tokens=1024, samples=[])
    assert report.tbt_attainment == 0.0
