"""Seeded engine scenarios shared by the oracle tests (CPU) and the device
parity tests (GPU).  Each case is a plain dict so it can also be rebuilt with
the reference's own dataclasses in oracle/make_golden.py."""
from __future__ import annotations

import random

import numpy as np


def case_params(seed: int) -> dict:
    """Randomised regime covering embedding, reserve draws, claims, deferral,
    swap/recompute, squeeze and collision preemptions (checked against the
    reference for seeds 0..59 during development)."""
    rnd = random.Random(seed)
    preset = rnd.choice(["alpaca", "sharegpt", "long"])
    if preset == "long":
        trace = dict(kind="spec", arrival_rate=rnd.choice([1.0, 2.0, 4.0]),
                     num_requests=rnd.choice([20, 40, 60]), input_mean=512, input_min=16,
                     input_max=4096, output_mean=1024, output_min=256, output_max=2048, length_cv=0.5)
    else:
        trace = dict(kind="preset", preset=preset, num_requests=rnd.choice([50, 150, 300]),
                     arrival_rate=rnd.choice([4.0, 16.0, 64.0]))
    slo = (rnd.choice([100_000, 500_000, 2_000_000]), rnd.choice([20_000, 60_000, 200_000]))
    bs = rnd.choice([4, 8, 16])
    cap = rnd.choice([1024, 2048, 4096, 8192]) // bs * bs
    if preset == "long":
        cap = max(cap, 6000 // bs * bs)
    truth = None if rnd.random() < 0.5 else dict(
        gamma_s=0.002, delta_s=8.0, alpha_r=1e-4, beta_r=rnd.choice([2.0, 1.7]), kappa_r=0.001, eps_r=0.5)
    pk = rnd.randrange(4)
    if pk == 0:
        pred = {}
    elif pk == 1:
        pred = dict(error_dist="uniform", error_scale=rnd.choice([24, 100]))
    elif pk == 2:
        pred = dict(error_dist="normal", error_scale=40, direction_accuracy=0.7)
    else:
        pred = dict(fixed_padding=rnd.choice([0, 5, 50]))
    reserved = rnd.choice([0, 2, 8])
    sched = dict(small_block_b=bs, victim_rule=rnd.choice(["slo", "slo", "fcfs"]),
                 token_budget=rnd.choice([512, 2048]), preallocate_m=rnd.choice([0, 2, 4]),
                 buffer_b=rnd.choice([2, 8]))
    fixed_conf = rnd.choice([None, None, 0.9])
    validate = rnd.choice([0, 1])
    return dict(seed=seed, trace=trace, slo=slo, capacity=cap, reserved=reserved, truth=truth,
                pred=pred, sched=sched, fixed_confidence=fixed_conf, validate_every=validate)


def build_product(params: dict):
    """(requests, EngineConfig) with the product's own host-side types."""
    import paper_2503_13773_b200 as P
    t = params["trace"]
    if t["kind"] == "preset":
        spec = P.PRESETS[t["preset"]].sized(t["num_requests"], t["arrival_rate"])
    elif t["kind"] == "spec":
        spec = P.TraceSpec(**{k: v for k, v in t.items() if k not in ("kind", "shard")})
    else:
        raise ValueError(t["kind"])
    seed = params["seed"]
    reqs = P.generate(spec, seed)
    P.assign_slos(reqs, params["slo"][0], params["slo"][1], P.SloPolicy(), seed)
    if "shard" in t:  # one instance's contiguous id range of a multi-instance trace
        reqs = reqs[t["shard"][0]:t["shard"][1]]
    tr = params["truth"]
    truth = P.TruthCosts.default() if tr is None else P.TruthCosts(
        P.SwapModel(tr["gamma_s"], tr["delta_s"]),
        P.RecomputeModel(tr["alpha_r"], tr["beta_r"], tr["kappa_r"], tr["eps_r"]))
    cfg = P.EngineConfig(
        capacity_tokens=params["capacity"], reserved_blocks=params["reserved"],
        sched=P.SchedulerConfig(**{"policy": "cacheopt", **params["sched"]}),
        predictor=P.PredictorConfig(**params["pred"]), truth=truth, seed=seed,
        fixed_confidence=params["fixed_confidence"], validate_every=params["validate_every"],
        record_events=params.get("record_events", True), allow_stacking=params.get("allow_stacking", False))
    return reqs, cfg


def config2(n: int = 65_536, seed: int = 0, capacity: int = 166_400, record_events: bool = True):
    """BASELINE.json config 2: ShareGPT-shaped, n requests arriving within
    ~n us, Llama-2-13B KV layout (16-token blocks), SLO baselines 2 s / 200 ms."""
    import paper_2503_13773_b200 as P
    spec = P.PRESETS["sharegpt"].sized(n, 1e6)
    reqs = P.generate(spec, seed)
    P.assign_slos(reqs, 2_000_000, 200_000, P.SloPolicy(), seed)
    cfg = P.EngineConfig(capacity_tokens=capacity, reserved_blocks=8,
                         sched=P.SchedulerConfig(small_block_b=16), seed=seed,
                         record_events=record_events)
    return reqs, cfg


def final_arrays(eng) -> dict:
    """Device engine per-request outcome arrays (sorted order) comparable with
    CacheOptOracle.final_state()."""
    f = eng._field
    return dict(
        state=f("STATE"), generated=f("GENERATED"), used=f("USED"), kv_need=f("KV_NEED"),
        prefill_done=f("PREFILL_DONE"), preemption_count=f("PREEMPTION_COUNT"),
        preemption_time_us=f("PREEMPTION_TIME"), first_token_at_us=f("FIRST_TOKEN"),
        last_token_at_us=f("LAST_TOKEN"), max_tbt_us=f("MAX_TBT"), ready_at_us=f("READY_AT"),
        first_start_us=f("FIRST_START"), completion_us=f("COMPLETION"), allocated_kvc=f("ALLOCATED_KVC"),
        predicted=f("PREDICTED"), estimated=f("ESTIMATED"), holds=f("HOLDS"),
        granted=np.where(f("HOLDS") == 1, f("GRANTED"), 0),
    )


# SLO baselines of BASELINE configs 1 and 3 from the reference's own
# calibrate_slo_baselines (engine.py:675-699, a vllm_block run), computed in
# the development container (tests/test_oracle_vs_reference_live.py re-derives them)
CONFIG1_SLO = (9141, 5070)
CONFIG3_SLO = (9674, 5140)


def config1(seed: int = 0, error: bool = False):
    """BASELINE config 1: ShareGPT 1K requests @4 req/s, OPT-13B-sized pool
    53,696 tokens, B = 8, reserve 8 blocks, CacheOPT; optionally the uniform
    +-24 predictor error used to exercise under-prediction."""
    import paper_2503_13773_b200 as P
    reqs = P.generate(P.PRESETS["sharegpt"].sized(1000, 4.0), seed)
    P.assign_slos(reqs, CONFIG1_SLO[0], CONFIG1_SLO[1], P.SloPolicy(), seed)
    pred = P.PredictorConfig(error_dist="uniform", error_scale=24) if error else P.PredictorConfig()
    cfg = P.EngineConfig(capacity_tokens=53_696, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=8),
                         predictor=pred, seed=seed)
    return reqs, cfg


def config3(seed: int = 0):
    """BASELINE config 3: the 2x-rate heavy-preemption regime (ShareGPT 1K @8
    req/s, 8,192-token pool, 16-token blocks)."""
    import paper_2503_13773_b200 as P
    reqs = P.generate(P.PRESETS["sharegpt"].sized(1000, 8.0), seed)
    P.assign_slos(reqs, CONFIG3_SLO[0], CONFIG3_SLO[1], P.SloPolicy(), seed)
    cfg = P.EngineConfig(capacity_tokens=8_192, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16),
                         seed=seed)
    return reqs, cfg
