"""The reference's pure scheduling-op and victim-ordering known answers
(pkg/tests/test_scheduler.py, pkg/tests/test_preemption.py) against the device
ops of paper_2503_13773_b200.scheduler (csrc/sched_ops.cuh: the planner's own
predicates, keys, compaction, rank sort and exact amortization).  Expected
values are the reference's; each test cites the one it restates."""
from fractions import Fraction

import numpy as np
import pytest

from paper_2503_13773_b200 import BucketConfig, Lifecycle
from paper_2503_13773_b200.scheduler import (AllocDemand, CriticalSets, PairCandidate, ReqView, VictimInfo,
                                             allocate_remaining, basic_demand, classify_critical, ensure_capacity,
                                             fill_token_budget, order_victims, pair_release, proactive_include,
                                             rlp_demand, s3_demand, victim_key)

pytestmark = pytest.mark.gpu
MS = 1_000
S = 1_000_000


def view(req_id=1, state=Lifecycle.WAITING, kv_need=10, generated=0, estimated_total=20, predicted_total=20,
         allocated=0, used=0, remaining_ttft_us=None, remaining_tbt_us=None, slo_tbt_us=200 * MS, arrival_us=0,
         ready=True):
    return ReqView(req_id=req_id, arrival_us=arrival_us, state=state, kv_need=kv_need, generated=generated,
                   estimated_total=estimated_total, predicted_total=predicted_total, allocated=allocated,
                   used=used, slo_ttft_us=500 * MS, slo_tbt_us=slo_tbt_us, remaining_ttft_us=remaining_ttft_us,
                   remaining_tbt_us=remaining_tbt_us, ready=ready)


def ids(vs):
    return [v.req_id for v in vs]


# -- criticality: test_scheduler.py:46-90 ----------------------------------------

def test_waiting_critical_iff_slack_below_epsilon(cuda_ok):
    sets = classify_critical([view(req_id=1, remaining_ttft_us=10 * MS), view(req_id=2, remaining_ttft_us=1000 * MS)],
                             [], t_i_max_us=50 * MS, epsilon_us=1 * MS)
    assert ids(sets.n_w) == [1] and ids(sets.n_w_prime) == [2]


def test_blown_deadlines_are_not_critical(cuda_ok):
    blown_tbt = view(req_id=3, state=Lifecycle.RUNNING, allocated=20, used=20, generated=5,
                     remaining_tbt_us=-5 * MS)
    sets = classify_critical([view(req_id=1, remaining_ttft_us=-5 * MS), view(req_id=2, remaining_ttft_us=-500)],
                             [blown_tbt], t_i_max_us=50 * MS, epsilon_us=1 * MS)
    assert ids(sets.n_w) == [2] and ids(sets.n_w_prime) == [1]
    assert sets.n_r == [] and ids(sets.n_r_prime) == [3]


def test_returned_spare_never_critical_and_exhausted_by_tbt(cuda_ok):
    spare = view(req_id=3, state=Lifecycle.RUNNING, allocated=40, used=20, generated=5, remaining_tbt_us=1 * MS)
    sets = classify_critical([], [spare], t_i_max_us=50 * MS, epsilon_us=1 * MS)
    assert sets.n_r == [] and sets.n_r_prime == []
    exhausted = view(req_id=4, state=Lifecycle.RUNNING, allocated=20, used=20, generated=5,
                     remaining_tbt_us=10 * MS)
    calm = view(req_id=5, state=Lifecycle.RUNNING, allocated=20, used=20, generated=5, remaining_tbt_us=2000 * MS)
    sets = classify_critical([], [exhausted, calm], t_i_max_us=50 * MS, epsilon_us=1 * MS)
    assert ids(sets.n_r) == [4] and ids(sets.n_r_prime) == [5]


def test_classify_orders_match_reference_keys(cuda_ok):
    # scheduler.py:151-162: n_w by (rt, id); n_w' by queue key (salvageable by
    # rt, then blown by arrival), ids breaking every tie; 700 views (> the
    # rank sort's shared-memory tile)
    rng = np.random.default_rng(5)
    vs = [view(req_id=int(i), remaining_ttft_us=int(rng.integers(-3, 4)) * 20 * MS,
               arrival_us=int(rng.integers(0, 5))) for i in rng.permutation(700)]
    sets = classify_critical(vs, [], t_i_max_us=50 * MS, epsilon_us=1 * MS)
    crit = [v for v in vs if -MS <= v.remaining_ttft_us and v.remaining_ttft_us - 50 * MS < MS]
    rest = [v for v in vs if v not in crit]
    assert ids(sets.n_w) == ids(sorted(crit, key=lambda v: (v.remaining_ttft_us, v.req_id)))
    qk = lambda v: (1, v.arrival_us, v.req_id) if v.remaining_ttft_us < 0 else (0, v.remaining_ttft_us, v.req_id)  # noqa: E731
    assert ids(sets.n_w_prime) == ids(sorted(rest, key=qk))


# -- demand: test_scheduler.py:93-117 (host arithmetic) -----------------------------

def test_demand_helpers(cuda_ok):
    n_w = [view(req_id=1, kv_need=40), view(req_id=2, kv_need=60)]
    n_r = [view(req_id=i, state=Lifecycle.RUNNING, allocated=8, used=8) for i in (3, 4, 5)]
    assert basic_demand(CriticalSets(n_w=n_w, n_r=n_r, n_w_prime=[], n_r_prime=[]), small_block_b=8) == 140
    assert basic_demand(CriticalSets([], [], [], []), 8) == 0
    assert basic_demand(CriticalSets([view(req_id=1, kv_need=40, allocated=30)], [], [], []), 8) == 18
    assert ensure_capacity(pool_free=100, d_kvc=140) == 40 and ensure_capacity(pool_free=200, d_kvc=140) == 0


# -- token budget: test_scheduler.py:123-150 ------------------------------------

def test_fill_token_budget(cuda_ok):
    q = [view(req_id=1, kv_need=40, remaining_ttft_us=50 * MS), view(req_id=2, kv_need=25, remaining_ttft_us=80 * MS)]
    sel, over = fill_token_budget(CriticalSets([], [], q, []), q, token_budget=100, consumed_tokens=30)
    assert ids(sel) == [1, 2] and not over
    q = [view(req_id=1, kv_need=60, remaining_ttft_us=50 * MS), view(req_id=2, kv_need=20, remaining_ttft_us=80 * MS)]
    sel, over = fill_token_budget(CriticalSets([], [], q, []), q, token_budget=100, consumed_tokens=50)
    assert sel == [] and not over
    sel, over = fill_token_budget(CriticalSets([], [], [], []), [], token_budget=100, consumed_tokens=130)
    assert sel == [] and over


# -- amortization: test_scheduler.py:155-230 ------------------------------------

def test_allocate_remaining_worked_examples(cuda_ok):
    assert allocate_remaining([AllocDemand(1, 30, 100, 30), AllocDemand(2, 40, 100, 10)], a_prime=100) == {1: 30, 2: 40}
    assert allocate_remaining([AllocDemand(1, 200, 100, 20), AllocDemand(2, 200, 100, 20)], a_prime=100) == \
        {1: 50, 2: 50}
    assert allocate_remaining([AllocDemand(1, 100, 2, 30), AllocDemand(2, 100, 1, 10)], a_prime=70) == {1: 60, 2: 10}
    g = allocate_remaining([AllocDemand(1, 100, -50, 30), AllocDemand(2, 100, 100, 30)], a_prime=50)
    assert sum(g.values()) == 50 and g[2] > g[1]
    with pytest.raises(ValueError):
        allocate_remaining([AllocDemand(1, 10, 1, 1)], a_prime=-1)


def _rational(demands, a_prime):
    wsum = sum(Fraction(max(1, d.rt_us)) * max(1, d.prompt_len) for d in demands)
    shares = {d.req_id: Fraction(a_prime) * Fraction(max(1, d.rt_us)) * max(1, d.prompt_len) / wsum for d in demands}
    floors = {i: int(s) for i, s in shares.items()}
    for i in sorted(shares, key=lambda i: (-(shares[i] - floors[i]), i))[:a_prime - sum(floors.values())]:
        floors[i] += 1
    return floors


@pytest.mark.parametrize("n_max", [9, 40, 600])  # warp path (<= 32), block path, block path past the smem tile
def test_allocate_remaining_sums_exactly_and_matches_rational_oracle(cuda_ok, n_max):
    # test_scheduler.py:174-201
    rng = np.random.default_rng(3)
    for _ in range(60 if n_max < 100 else 8):
        n = int(rng.integers(1, n_max))
        demands = [AllocDemand(int(i), int(rng.integers(1, 500)), int(rng.integers(1, 10_000_000)),
                               int(rng.integers(1, 3000))) for i in rng.permutation(n)]
        a_prime = int(rng.integers(0, sum(d.m_tokens for d in demands)))
        grants = allocate_remaining(demands, a_prime=a_prime)
        assert sum(grants.values()) == a_prime
        assert grants == _rational(demands, a_prime)


def _rational_inverted(demands, a_prime):
    # scheduler.py:229-243 with invert=True (weights 1/(rt*p), :233)
    live = [d for d in demands if d.m_tokens > 0]
    if sum(d.m_tokens for d in live) <= a_prime:
        return {d.req_id: d.m_tokens for d in live}
    w = {d.req_id: 1 / Fraction(max(1, d.rt_us) * max(1, d.prompt_len)) for d in live}
    wsum = sum(w.values())
    shares = {i: Fraction(a_prime) * x / wsum for i, x in w.items()}
    floors = {i: int(s) for i, s in shares.items()}
    for i in sorted(shares, key=lambda i: (-(shares[i] - floors[i]), i))[:a_prime - sum(floors.values())]:
        floors[i] += 1
    return floors


@pytest.mark.parametrize("n_max", [9, 40, 300])
def test_allocate_remaining_inverted_matches_rational_oracle(cuda_ok, n_max):
    # exact multi-precision path (planner.cuh amortize_inverted)
    rng = np.random.default_rng(5)
    for t in range(40 if n_max < 100 else 6):
        n = int(rng.integers(1, n_max))
        hi = [10, 1000, 10_000_000][t % 3]  # small weight ranges force duplicate weights and exact ties
        demands = [AllocDemand(int(i), int(rng.integers(0, 500)), int(rng.integers(-5, hi)),
                               int(rng.integers(1, 3000 if hi > 10 else 4))) for i in rng.permutation(n)]
        a_prime = int(rng.integers(0, max(1, sum(d.m_tokens for d in demands))))
        grants = allocate_remaining(demands, a_prime=a_prime, invert=True)
        assert grants == _rational_inverted(demands, a_prime)


def test_allocate_remaining_inverted_exact_ties_and_wide_weights(cuda_ok):
    # equal weights with m | a': integer shares, no remainder; equal weights
    # otherwise: ties broken by id; weights near 2^62 (rt*p wide)
    same = [AllocDemand(i, 100, 50, 4) for i in (5, 2, 9, 7)]
    assert allocate_remaining(same, a_prime=80, invert=True) == {5: 20, 2: 20, 9: 20, 7: 20}
    assert allocate_remaining(same, a_prime=82, invert=True) == _rational_inverted(same, 82) == \
        {5: 21, 2: 21, 9: 20, 7: 20}
    # w = 1 and w = 2: shares 2/3 a' and 1/3 a'
    pair = [AllocDemand(1, 1000, 1, 1), AllocDemand(2, 1000, 2, 1), AllocDemand(3, 1000, 2, 1)]
    for a in (0, 1, 2, 3, 4, 5, 99, 100, 101):
        assert allocate_remaining(pair, a_prime=a, invert=True) == _rational_inverted(pair, a), a
    wide = [AllocDemand(i, 10**6, (1 << 40) + 977 * i, (1 << 22) - i) for i in range(12)]
    assert allocate_remaining(wide, a_prime=777_777, invert=True) == _rational_inverted(wide, 777_777)


def test_allocate_remaining_rt_scaling_invariance(cuda_ok):
    # test_scheduler.py:204-219
    rng = np.random.default_rng(4)
    for _ in range(30):
        n = int(rng.integers(2, 7))
        demands = [AllocDemand(i, int(rng.integers(1, 300)), int(rng.integers(1, 1_000_000)),
                               int(rng.integers(1, 500))) for i in range(n)]
        a_prime = max(0, sum(d.m_tokens for d in demands) - 17)
        scaled = [AllocDemand(d.req_id, d.m_tokens, d.rt_us * 7, d.prompt_len) for d in demands]
        assert allocate_remaining(scaled, a_prime=a_prime) == allocate_remaining(demands, a_prime=a_prime)


# -- pair release / proactive: test_scheduler.py:233-273 --------------------------

def test_pair_release(cuda_ok):
    assert pair_release(150, 12, [PairCandidate(9, 10, 200)]) == 9
    assert pair_release(150, 12, [PairCandidate(9, 10, 100)]) is None
    assert pair_release(150, 12, [PairCandidate(9, 15, 300)]) is None
    assert pair_release(150, 12, [PairCandidate(9, 10, 200), PairCandidate(3, 4, 200), PairCandidate(5, 4, 200)]) == 3
    assert pair_release(150, 12, []) is None


def test_proactive_include_boundary(cuda_ok):
    soon = view(req_id=1, state=Lifecycle.RUNNING, kv_need=10, generated=18, estimated_total=20, allocated=29, used=28)
    later = view(req_id=2, state=Lifecycle.RUNNING, kv_need=10, generated=17, estimated_total=20, allocated=29,
                 used=27)
    full = view(req_id=3, state=Lifecycle.RUNNING, kv_need=10, generated=18, estimated_total=20, allocated=30, used=28)
    assert ids(proactive_include([soon, later, full], m=2)) == [1]


def test_baseline_demands(cuda_ok):
    # test_scheduler.py:276-284
    assert s3_demand(130, bucket_tokens=50, preempt_count=0) == 150
    assert s3_demand(130, bucket_tokens=50, preempt_count=1) == 300
    assert s3_demand(50, bucket_tokens=50, preempt_count=0) == 50
    assert rlp_demand(60, padding=100) == 160 and rlp_demand(0, padding=100) == 101


# -- victim ordering: test_preemption.py:39-105 ----------------------------------

def vi(req_id, slo_s, remaining, occupancy):
    return VictimInfo(req_id=req_id, slo_tbt_us=int(slo_s * S), remaining_tokens=remaining, occupancy_tokens=occupancy)


def test_victim_order_known_answers(cuda_ok):
    cfg = BucketConfig()
    assert ids(order_victims([vi(1, 0.6, 200, 300), vi(2, 0.3, 500, 100), vi(3, 1.0, 400, 150)], cfg)) == [3, 1, 2]
    assert ids(order_victims([vi(1, 0.6, 200, 200), vi(2, 0.6, 200, 100)], cfg)) == [2, 1]
    assert ids(order_victims([vi(5, 0.1, 10, 10)], cfg)) == [5] and order_victims([], cfg) == []
    assert ids(order_victims([vi(9, 0.6, 200, 100), vi(4, 0.6, 200, 100)], cfg)) == [4, 9]
    lo, mid, top = (victim_key(int(x * S), 0, 1, 0, cfg) for x in (0.01, 0.1, 5.0))
    assert top < mid < lo


def test_victim_order_permutation_stable_and_matches_keys(cuda_ok):
    # test_preemption.py:67-81, plus equality with the reference key order
    rng = np.random.default_rng(11)
    cfg = BucketConfig()
    for _ in range(40):
        n = int(rng.integers(1, 40))
        infos = [vi(i, float(rng.uniform(0.01, 3.0)), int(rng.integers(0, 900)), int(rng.integers(1, 900)))
                 for i in range(n)]
        want = ids(sorted(infos, key=lambda v: victim_key(v.slo_tbt_us, v.remaining_tokens, v.occupancy_tokens,
                                                          v.req_id, cfg)))
        for _ in range(3):
            perm = list(infos)
            rng.shuffle(perm)
            assert ids(order_victims(perm, cfg)) == want
