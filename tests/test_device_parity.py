"""Device engine vs the CPU oracle on seeded traces: event logs, per-request
outcomes and pool totals must be bit-identical (integer decisions)."""
import numpy as np
import pytest

from oracle.cacheopt_oracle import CacheOptOracle
from tests.cases import build_product, case_params, config2, final_arrays

pytestmark = pytest.mark.gpu


def _compare(eng, orc, label):
    ev_d, ev_o = eng.events, orc.events
    if ev_d != ev_o:
        for k, (a, b) in enumerate(zip(ev_d, ev_o)):
            if a != b:
                raise AssertionError(f"{label}: first event diff at {k}:\n dev {a}\n orc {b}")
        raise AssertionError(f"{label}: event count {len(ev_d)} vs {len(ev_o)}")
    fo = orc.final_state()
    fd = final_arrays(eng)
    for k, v in fd.items():
        assert np.array_equal(np.asarray(v), np.asarray(fo[k])), f"{label}: field {k} differs"
    s = eng._scalars()
    assert s.footprint_tokens == orc.fp_sum and s.used_tokens == orc.used_sum
    assert s.reserved_blocks_current == orc.rsv_cur
    assert eng.samples == orc.samples
    # N1: identical physical block tables and free stack
    assert eng.block_tables() == orc.block_tables(), f"{label}: block tables differ"


@pytest.mark.parametrize("seed", list(range(0, 48)))
def test_random_regimes_full_run(cuda_ok, seed):
    from paper_2503_13773_b200 import Engine
    reqs, cfg = build_product(case_params(seed))
    eng = Engine(reqs, cfg)
    eng.run_steps(0)
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    _compare(eng, orc, f"seed {seed}")
    eng.close()


@pytest.mark.parametrize("seed", [3, 7])
def test_step_api_matches_run(cuda_ok, seed):
    from paper_2503_13773_b200 import Engine
    reqs, cfg = build_product(case_params(seed))
    eng = Engine(reqs, cfg)
    n = 0
    while eng.step():
        n += 1
        assert n < 200_000
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    _compare(eng, orc, f"step seed {seed}")


def test_config2_first_60_steps(cuda_ok):
    from paper_2503_13773_b200 import Engine
    reqs, cfg = config2(n=65_536)
    eng = Engine(reqs, cfg)
    eng.run_steps(60)
    orc = CacheOptOracle(reqs, cfg)
    for _ in range(60):
        orc.step()
    _compare(eng, orc, "config2")


@pytest.mark.parametrize("seed,drain", [(4, True), (8, True), (4, False)])
def test_step_result_members_match_iter_events(cuda_ok, seed, drain):
    # the (req_id, tokens) pairs the library writes per step (co_step_args
    # ids / members_ids) against the iter events, with and without the drain
    from paper_2503_13773_b200 import Engine
    reqs, cfg = build_product(case_params(seed))
    eng = Engine(reqs, cfg)
    got = []
    while True:
        more, members, end = eng.step_result(drain=drain)
        if len(members):
            got.append((end, members.tolist()))
        if not more:
            break
    iters = [(e["end"], e["members"]) for e in eng.events if e["ev"] == "iter"]
    assert got == iters
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    assert eng.events == orc.events


@pytest.mark.parametrize("which", ["config1", "config1_err", "config3"])
def test_baseline_configs_full_run(cuda_ok, which):
    """BASELINE.json configs 1 and 3 end to end (tens of thousands of steps)."""
    from paper_2503_13773_b200 import Engine
    from tests.cases import config1, config3
    reqs, cfg = {"config1": lambda: config1(), "config1_err": lambda: config1(error=True),
                 "config3": lambda: config3()}[which]()
    eng = Engine(reqs, cfg, steps_per_launch=64)
    eng.run_steps(0)
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    _compare(eng, orc, which)


# allow_stacking=True (kvc.py:187-192, :212, :263-270): hosts carry several
# guests (up to 4 at once in these regimes); the oracle's stacking is pinned
# to the reference by tests/golden/stack_case* and the live cross-check
@pytest.mark.parametrize("seed", [3, 8, 13, 14, 15, 21, 49, 57])
def test_stacking_regimes_full_run(cuda_ok, seed):
    from paper_2503_13773_b200 import Engine
    p = case_params(seed)
    p["allow_stacking"] = True
    reqs, cfg = build_product(p)
    eng = Engine(reqs, cfg)
    eng.run_steps(0)
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    _compare(eng, orc, f"stacking seed {seed}")
    eng.close()


@pytest.mark.parametrize("seed", [8, 13])
def test_stacking_guest_lists_every_step(cuda_ok, seed):
    # the pool's guest lists (embed order) and offsets after every step
    from paper_2503_13773_b200 import Engine
    p = case_params(seed)
    p["allow_stacking"] = True
    reqs, cfg = build_product(p)
    eng = Engine(reqs, cfg)
    orc = CacheOptOracle(reqs, cfg)
    most = 0
    while True:
        more = eng.step()
        orc.step()
        want = {orc.rid[h]: [orc.rid[g] for g in gl] for h, gl in orc.guests.items() if gl}
        got = {r: eng.pool.guests_of(r) for r in want}
        assert got == want
        most = max([most] + [len(v) for v in want.values()])
        if not more:
            break
    assert most >= 3


# invert_amortization=True (scheduler.py:43, :229-243 with weights 1/(rt*p),
# :233): the exact multi-precision amortization (planner.cuh
# amortize_inverted); the oracle's Fraction restatement is pinned to the
# reference by tests/golden/inv_case* and the live cross-check
@pytest.mark.parametrize("seed", [0, 5, 6, 7, 9, 11, 12, 15, 16, 18, 20, 25, 29])
def test_inverted_amortization_full_run(cuda_ok, seed):
    from paper_2503_13773_b200 import Engine
    p = case_params(seed)
    p["sched"] = {**p["sched"], "invert_amortization": True}
    reqs, cfg = build_product(p)
    eng = Engine(reqs, cfg)
    eng.run_steps(0)
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    _compare(eng, orc, f"inverted amortization seed {seed}")
    eng.close()


@pytest.mark.parametrize("seed", [8, 13])
def test_inverted_amortization_with_stacking(cuda_ok, seed):
    from paper_2503_13773_b200 import Engine
    p = case_params(seed)
    p["sched"] = {**p["sched"], "invert_amortization": True}
    p["allow_stacking"] = True
    reqs, cfg = build_product(p)
    eng = Engine(reqs, cfg)
    eng.run_steps(0)
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    _compare(eng, orc, f"inverted amortization + stacking seed {seed}")
    eng.close()
