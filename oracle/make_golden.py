"""Generates tests/golden/ from the UNMODIFIED reference simulator.

Run in the development container (where /root/reference exists):

    python oracle/make_golden.py

For every scenario of tests/cases.py (and a config-2 window) it builds the
trace and config with the reference's OWN classes (kvcsim.workload.generate,
assign_slos, EngineConfig, ...), runs kvcsim.engine.Engine, and stores the
trace columns, the config parameters, the full event log (gzip'd sorted-key
JSONL, exactly write_events_jsonl's bytes) and per-request final outcomes.
The oracle is pinned against these files by tests/test_oracle_golden.py; the
device engine is checked against the oracle on the GPU.
"""
from __future__ import annotations

import copy
import gzip
import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)

SEEDS = [0, 1, 2, 5, 9, 13, 21, 34]
STACK_SEEDS = [8, 13, 57]
INVERT_SEEDS = [7, 9, 12, 18]  # invert_amortization=True (scheduler.py:43, :233): grants differ from the default  # regimes where a host carries up to 3-4 stacked guests (allow_stacking=True)
BASELINE_CASES = [("vllm_block", 5), ("vllm_block", 13), ("sarathi_chunked", 13), ("sarathi_chunked", 9),
                  ("rlp", 6), ("s3", 2), ("s3", 13)]


def ref_build(params):
    sys.path.insert(0, REF)
    from kvcsim.costmodel import TruthCosts
    from kvcsim.engine import EngineConfig
    from kvcsim.estimation import PredictorConfig
    from kvcsim.preemption import RecomputeModel, SwapModel
    from kvcsim.scheduler import SchedulerConfig
    from kvcsim.workload import PRESETS, SloPolicy, TraceSpec, assign_slos, generate
    t = params["trace"]
    if t["kind"] == "preset":
        spec = PRESETS[t["preset"]].sized(t["num_requests"], t["arrival_rate"])
    else:
        spec = TraceSpec(**{k: v for k, v in t.items() if k not in ("kind", "shard")})
    seed = params["seed"]
    reqs = generate(spec, seed)
    assign_slos(reqs, params["slo"][0], params["slo"][1], SloPolicy(), seed)
    if "shard" in t:  # BASELINE config 4: one instance's contiguous id range
        reqs = reqs[t["shard"][0]:t["shard"][1]]
    tr = params["truth"]
    truth = TruthCosts.default() if tr is None else TruthCosts(
        swap_true=SwapModel(tr["gamma_s"], tr["delta_s"]),
        recompute_true=RecomputeModel(tr["alpha_r"], tr["beta_r"], tr["kappa_r"], tr["eps_r"]))
    cfg = EngineConfig(capacity_tokens=params["capacity"], reserved_blocks=params["reserved"],
                       sched=SchedulerConfig(**{"policy": "cacheopt", **params["sched"]}),
                       predictor=PredictorConfig(**params["pred"]), truth=truth, seed=seed,
                       fixed_confidence=params["fixed_confidence"],
                       validate_every=params["validate_every"],
                       allow_stacking=params.get("allow_stacking", False))
    return reqs, cfg


def jsonl_bytes(events) -> bytes:
    return "".join(json.dumps(e, sort_keys=True, separators=(",", ":")) + "\n" for e in events).encode()


TRACE_COLS = ("id", "arrival_us", "prompt_len", "true_output_len", "slo_ttft_us", "slo_tbt_us")


def trace_digest(cols) -> str:
    h = hashlib.sha256()
    for k in TRACE_COLS:
        h.update(np.asarray(cols[k], dtype=np.int64).tobytes())
    return h.hexdigest()


def run_and_store(name, params, reqs, cfg, steps=None, keep_events=True, store_trace=True):
    from kvcsim.engine import Engine
    trace = {k: [getattr(r, k) for r in reqs] for k in TRACE_COLS}
    digest = trace_digest(trace)
    if not store_trace:
        trace = None
    eng = Engine(copy.deepcopy(reqs), cfg)
    metrics = None
    if steps is None:
        metrics = eng.run().to_dict()  # engine.py:643-672: the reference's own MetricsReport
    else:
        for _ in range(steps):
            eng.step()
    blob = jsonl_bytes(eng.events)
    order = sorted(range(len(reqs)), key=lambda k: (reqs[k].arrival_us, reqs[k].id))
    final = {}
    for f in ("generated", "preemption_count", "preemption_time_us", "max_tbt_us", "kv_need", "prefill_done"):
        final[f] = [getattr(eng.runtimes[reqs[k].id], f) for k in order]
    final["used"] = [eng.runtimes[reqs[k].id].used_kvc for k in order]
    final["completion_us"] = [eng.runtimes[reqs[k].id].completion_us or -1 for k in order]
    final["first_token_at_us"] = [
        -1 if eng.runtimes[reqs[k].id].first_token_at_us is None else eng.runtimes[reqs[k].id].first_token_at_us
        for k in order]
    doc = {"name": name, "params": params, "steps": steps, "trace": trace, "trace_sha256": digest,
           "events_sha256": hashlib.sha256(blob).hexdigest(), "n_events": len(eng.events),
           "final": final, "pool": {"footprint": eng.pool.footprint_tokens, "used": eng.pool.used_tokens,
                                    "reserved": eng.pool.reserved_blocks_current},
           "samples_sha256": hashlib.sha256(json.dumps(eng._samples).encode()).hexdigest(),
           "metrics": metrics}
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, name + ".json.gz"), "wb") as raw, \
            gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as fh:  # reproducible bytes
        fh.write(json.dumps(doc).encode())
    if keep_events:
        with open(os.path.join(OUT, name + ".events.jsonl.gz"), "wb") as raw, \
                gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as fh:
            fh.write(blob)
    print(f"{name}: {len(eng.events)} events sha={doc['events_sha256'][:12]}")


def main():
    sys.path.insert(0, REF)
    from tests.cases import case_params
    only = set(sys.argv[1:])
    for s in SEEDS:
        if only and f"case{s:02d}" not in only:
            continue
        p = case_params(s)
        reqs, cfg = ref_build(p)
        run_and_store(f"case{s:02d}", p, reqs, cfg)
    # allow_stacking=True (kvc.py:187-192, :212): several guests per host
    for s in STACK_SEEDS:
        name = f"stack_case{s:02d}"
        if only and name not in only:
            continue
        p = case_params(s)
        p["allow_stacking"] = True
        reqs, cfg = ref_build(p)
        run_and_store(name, p, reqs, cfg)
    # invert_amortization=True: amortization weights 1/(rt*p) (scheduler.py:233)
    for s in INVERT_SEEDS:
        name = f"inv_case{s:02d}"
        if only and name not in only:
            continue
        p = case_params(s)
        p["sched"] = {**p["sched"], "invert_amortization": True}
        reqs, cfg = ref_build(p)
        run_and_store(name, p, reqs, cfg)
    # the four baseline planners (scheduler.py:760-936) on regimes that preempt
    for pol, s in BASELINE_CASES:
        name = f"base_{pol}_case{s:02d}"
        if only and name not in only:
            continue
        p = case_params(s)
        p["sched"] = {**p["sched"], "policy": pol}
        reqs, cfg = ref_build(p)
        run_and_store(name, p, reqs, cfg)
    # config 2 window: 65,536 requests, first 60 steps (digest + final state only)
    if only and not only & {"config2_60", "config1", "config3", "config5", "config4_shard1_60",
                            "config4_shard7_60"}:
        return
    p = {"seed": 0, "trace": {"kind": "preset", "preset": "sharegpt", "num_requests": 65536,
                               "arrival_rate": 1e6},
         "slo": [2_000_000, 200_000], "capacity": 166_400, "reserved": 8, "truth": None, "pred": {},
         "sched": {"small_block_b": 16}, "fixed_confidence": None, "validate_every": 0}
    if not only or "config2_60" in only:
        reqs, cfg = ref_build(p)
        run_and_store("config2_60", p, reqs, cfg, steps=60, keep_events=False, store_trace=False)
    # BASELINE config 4: shards 1 and 7 of the 8 x 65,536-request trace (the
    # bench's make_trace(rank, 8)), first 60 steps each
    for r in (1, 7):
        name = f"config4_shard{r}_60"
        if only and name not in only:
            continue
        p = {"seed": 0, "trace": {"kind": "preset", "preset": "sharegpt", "num_requests": 8 * 65536,
                                   "arrival_rate": 8e6, "shard": [r * 65536, (r + 1) * 65536]},
             "slo": [2_000_000, 200_000], "capacity": 166_400, "reserved": 8, "truth": None, "pred": {},
             "sched": {"small_block_b": 16}, "fixed_confidence": None, "validate_every": 0}
        reqs, cfg = ref_build(p)
        run_and_store(name, p, reqs, cfg, steps=60, keep_events=False, store_trace=False)
    # BASELINE config 5: the 200-request long-output trace (the bench's decode
    # leg, bench.long_output_trace), 65,536-token pool, full run
    if not only or "config5" in only:
        p = {"seed": 0, "trace": {"kind": "spec", "arrival_rate": 1.0, "num_requests": 200, "input_mean": 512,
                                   "input_min": 16, "input_max": 4096, "output_mean": 4096, "output_min": 1024,
                                   "output_max": 8192, "length_cv": 0.5},
             "slo": [2_000_000, 100_000], "capacity": 65_536, "reserved": 8, "truth": None, "pred": {},
             "sched": {"small_block_b": 16}, "fixed_confidence": None, "validate_every": 0}
        reqs, cfg = ref_build(p)
        run_and_store("config5", p, reqs, cfg, keep_events=False, store_trace=False)
    if only and not only & {"config1", "config3"}:
        return
    # BASELINE configs 1 and 3, full runs, with the reference's own calibrated SLO baselines
    from tests.cases import CONFIG1_SLO, CONFIG3_SLO
    for name, rate, cap, bs, slo in (("config1", 4.0, 53_696, 8, CONFIG1_SLO), ("config3", 8.0, 8_192, 16, CONFIG3_SLO)):
        p = {"seed": 0, "trace": {"kind": "preset", "preset": "sharegpt", "num_requests": 1000, "arrival_rate": rate},
             "slo": list(slo), "capacity": cap, "reserved": 8, "truth": None, "pred": {},
             "sched": {"small_block_b": bs}, "fixed_confidence": None, "validate_every": 0}
        reqs, cfg = ref_build(p)
        run_and_store(name, p, reqs, cfg, keep_events=False, store_trace=False)


if __name__ == "__main__":
    main()
