"""Row (f).1: compute_metrics on the device.  CPU: the host half (percentile
interpolation from selected order statistics) equals np.percentile exactly.
GPU: Engine.run()'s device-aggregated report equals report_host() (the
reference definition over host views)
field for field (exact float equality) across randomized regimes and the
BASELINE configs."""
import numpy as np
import pytest

from paper_2503_13773_b200.engine import _pct, order_stat_ranks, pct_from_order_stats


@pytest.mark.parametrize("seed", range(12))
def test_percentiles_from_order_stats_match_numpy(seed):
    rng = np.random.default_rng(seed)
    for n in [1, 2, 3, 7, 10, 99, 100, 101, 1000, 12345]:
        if seed % 2:
            vals = rng.integers(0, 10**7, n).astype(float)
            total = int(vals.sum())
        else:
            vals = rng.random(n) * 1e4
            total = float(np.add.reduce(vals))
        srt = np.sort(vals)
        os7 = [srt[k] for k in order_stat_ranks(n)]
        assert pct_from_order_stats(n, os7, total) == _pct(list(vals))


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["case0", "case1", "case2", "case5", "case9", "case13", "config1", "config3"])
def test_device_report_equals_host_report(cuda_ok, which):
    import paper_2503_13773_b200 as P
    from tests.cases import build_product, case_params, config1, config3
    if which.startswith("case"):
        reqs, cfg = build_product(case_params(int(which[4:])))
    else:
        reqs, cfg = (config1 if which == "config1" else config3)()
    eng = P.Engine(reqs, cfg)
    dev = eng.run()  # run() aggregates on the device
    host = eng.report_host()
    assert dev.to_dict() == host.to_dict()
    eng.close()
