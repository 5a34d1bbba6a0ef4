"""When the reference is present (development container), run it side by
side with the oracle on more randomised regimes than the fixtures hold."""
import copy
import sys

import pytest

from tests.conftest import REFERENCE_SRC, has_reference

pytestmark = [pytest.mark.reference,
              pytest.mark.skipif(not has_reference(), reason="reference not mounted")]


@pytest.mark.parametrize("seed", [40, 41, 42, 43, 44, 45])
def test_oracle_matches_live_reference(seed):
    sys.path.insert(0, REFERENCE_SRC)
    from kvcsim.engine import Engine
    from oracle.cacheopt_oracle import CacheOptOracle
    from oracle.make_golden import ref_build
    from tests.cases import case_params
    reqs, cfg = ref_build(case_params(seed))
    eng = Engine(copy.deepcopy(reqs), cfg)
    eng.run()
    orc = CacheOptOracle(reqs, cfg)   # the oracle accepts the reference's own config objects
    orc.run()
    assert orc.events == eng.events
    for k, rid in enumerate(orc.rid):
        assert orc.token_times[k] == eng.runtimes[rid].token_times_us


@pytest.mark.parametrize("seed", [3, 14, 15, 21, 49])
def test_oracle_matches_live_reference_with_stacking(seed):
    # allow_stacking=True (kvc.py:187-192, :212, :263-270): hosts carry several guests
    sys.path.insert(0, REFERENCE_SRC)
    from kvcsim.engine import Engine
    from oracle.cacheopt_oracle import CacheOptOracle
    from oracle.make_golden import ref_build
    from tests.cases import case_params
    p = case_params(seed)
    p["allow_stacking"] = True
    reqs, cfg = ref_build(p)
    eng = Engine(copy.deepcopy(reqs), cfg)
    eng.run()
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    assert orc.events == eng.events


def test_config_slo_baselines_match_reference_calibration():
    import copy
    sys.path.insert(0, REFERENCE_SRC)
    from kvcsim.engine import EngineConfig, calibrate_slo_baselines
    from kvcsim.scheduler import SchedulerConfig
    from kvcsim.workload import PRESETS, generate
    from tests.cases import CONFIG1_SLO
    reqs = generate(PRESETS["sharegpt"].sized(1000, 4.0), 0)
    cfg = EngineConfig(capacity_tokens=53_696, reserved_blocks=8, sched=SchedulerConfig(small_block_b=8), seed=0)
    assert calibrate_slo_baselines(copy.deepcopy(reqs), cfg) == CONFIG1_SLO


@pytest.mark.parametrize("seed", [0, 6, 11, 16])
def test_oracle_matches_live_reference_inverted_amortization(seed):
    # invert_amortization=True: weights 1/(rt*p) (scheduler.py:233)
    sys.path.insert(0, REFERENCE_SRC)
    from kvcsim.engine import Engine
    from oracle.cacheopt_oracle import CacheOptOracle
    from oracle.make_golden import ref_build
    from tests.cases import case_params
    p = case_params(seed)
    p["sched"] = {**p["sched"], "invert_amortization": True}
    reqs, cfg = ref_build(p)
    eng = Engine(copy.deepcopy(reqs), cfg)
    eng.run()
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    assert orc.events == eng.events
