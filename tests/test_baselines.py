"""Row (f).2: the reference's baseline planners (scheduler.py:760-936:
vllm_block, sarathi_chunked, rlp, s3) on the device.  The oracle's
restatement is pinned to golden logs of the unmodified reference
(tests/golden/base_*, via test_oracle_golden); here the device engine must
reproduce the oracle's event logs, per-request outcomes and block tables
bit for bit, and a device SLO calibration run (engine.py:675-699 runs
vllm_block) must match the reference's calibrated baselines."""
import dataclasses

import numpy as np
import pytest

from oracle.cacheopt_oracle import CacheOptOracle
from tests.cases import build_product, case_params, final_arrays

POLICIES = ["vllm_block", "sarathi_chunked", "rlp", "s3"]


def _with_policy(cfg, pol):
    return dataclasses.replace(cfg, sched=dataclasses.replace(cfg.sched, policy=pol))


@pytest.mark.gpu
@pytest.mark.parametrize("pol", POLICIES)
@pytest.mark.parametrize("seed", [0, 2, 5, 6, 9, 13])
def test_device_baseline_matches_oracle(cuda_ok, pol, seed):
    import paper_2503_13773_b200 as P
    reqs, cfg = build_product(case_params(seed))
    cfg = _with_policy(cfg, pol)
    eng = P.Engine(reqs, cfg)
    eng.run_steps(0)
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    assert eng.events == orc.events
    fo = orc.final_state()
    for k, v in final_arrays(eng).items():
        assert np.array_equal(v, fo[k]), k
    assert eng.block_tables() == orc.block_tables()
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("pol", POLICIES)
def test_device_baselines_on_baseline_config3(cuda_ok, pol):
    import paper_2503_13773_b200 as P
    from tests.cases import config3
    reqs, cfg = config3()
    cfg = _with_policy(cfg, pol)
    eng = P.Engine(reqs, cfg)
    rep = eng.run()
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    assert eng.events == orc.events
    assert rep.to_dict() == eng.report_host().to_dict()
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("which", ["config1", "config3"])
def test_device_slo_calibration_matches_reference(cuda_ok, which):
    # engine.py:675-699 on the device (a vllm_block run); the expected pairs
    # are the reference's own calibration (tests/cases.py CONFIG*_SLO,
    # re-derived live by test_oracle_vs_reference_live)
    import paper_2503_13773_b200 as P
    from tests.cases import CONFIG1_SLO, CONFIG3_SLO
    rate, cap, bs, want = (4.0, 53_696, 8, CONFIG1_SLO) if which == "config1" else (8.0, 8_192, 16, CONFIG3_SLO)
    reqs = P.generate(P.PRESETS["sharegpt"].sized(1000, rate), 0)
    cfg = P.EngineConfig(capacity_tokens=cap, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=bs), seed=0)
    assert P.calibrate_slo_baselines(reqs, cfg) == want
