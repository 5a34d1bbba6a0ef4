"""Host-side float evaluation and exact integer restatements against the
reference's known-answer tests."""
import math
import random
from fractions import Fraction


import paper_2503_13773_b200 as P
from oracle.cacheopt_oracle import split_largest_remainder
from paper_2503_13773_b200 import hostprep as H


def test_padding_known_answers():
    # test_estimation.py:28-39 (range 1000 at c=0.9 caps at the range; c=0.5 -> 589)
    cfg = P.EngineConfig(predictor=P.PredictorConfig(bin_width=1001))
    assert H.run_padding(cfg, 0.9) == 1000
    assert H.run_padding(cfg, 0.5) == math.floor(1000 * math.sqrt(-math.log(0.5) / 2) + 0.5)
    assert H.run_padding(P.EngineConfig(predictor=P.PredictorConfig(bin_width=1)), 0.9) == 0
    assert H.run_padding(P.EngineConfig(predictor=P.PredictorConfig(fixed_padding=25)), 0.9) == 25
    # default bin 50 at the clamped confidence 0.5
    assert H.run_padding(P.EngineConfig(), 0.5) == 29


def test_confidence_clamps_like_the_reference():
    cfg = P.EngineConfig()
    import numpy as np
    assert H.run_confidence(cfg, np.array([0, 1_000_000])) == 0.5
    assert H.run_confidence(P.EngineConfig(fixed_confidence=0.9), np.array([0])) == 0.9


def test_sweet_spot_default_is_4000():
    tc = P.TruthCosts.default()
    assert abs(H.sweet_spot(tc.swap_true, tc.recompute_true) - 4000) <= 1  # test_preemption.py:180-183


def test_charge_luts_match_to_us():
    cfg = P.EngineConfig()
    half, rec, ss, sr = H.charge_luts(cfg, 5000)
    tc = cfg.truth
    for s in (1, 7, 1000, 4000, 4001, 5000):
        assert half[s] == P.to_us(tc.swap_true.predict(s) / 2.0)
        assert rec[s] == P.to_us(tc.recompute_true.predict(s))
        assert ss[s] == int(tc.swap_true.predict(s) * 1000 + 0.5)


def _fraction_split(demands, a):
    # the reference's rational construction (scheduler.py:229-243), restated
    live = [d for d in demands if d[1] > 0]
    if sum(d[1] for d in live) <= a:
        return {d[0]: d[1] for d in live}
    w = {d[0]: Fraction(max(1, d[2]) * max(1, d[3])) for d in live}
    W = sum(w.values())
    sh = {k: Fraction(a) * v / W for k, v in w.items()}
    g = {k: int(v) for k, v in sh.items()}
    left = a - sum(g.values())
    for k in sorted(sh, key=lambda k: (-(sh[k] - g[k]), k))[:left]:
        g[k] += 1
    return g


def test_integer_split_equals_rational_oracle():
    rng = random.Random(7)
    for _ in range(300):
        n = rng.randint(1, 12)
        demands = [(rng.randint(0, 10**6), rng.randint(-5, 500), rng.randint(-10, 10**9), rng.randint(0, 4000))
                   for _ in range(n)]
        ids = set()
        demands = [d for d in demands if not (d[0] in ids or ids.add(d[0]))]
        a = rng.randint(0, 2000)
        assert split_largest_remainder(demands, a) == _fraction_split(demands, a)


def test_worked_amortization_example():
    # test_scheduler.py:167-171 shape: weights 6:1 over 70 tokens -> [60, 10]
    g = split_largest_remainder([(1, 100, 6, 1), (2, 100, 1, 1)], 70)
    assert g == {1: 60, 2: 10}


def test_workload_matches_reference_presets():
    spec = P.PRESETS["sharegpt"]
    assert (spec.input_mean, spec.output_mean, spec.input_max, spec.output_max) == (161.31, 337.99, 3200, 991)
    reqs = P.generate(spec.sized(50, 4.0), 3)
    assert [r.id for r in reqs] == list(range(50))
    assert all(16 <= r.prompt_len <= 3200 for r in reqs)
