"""Generates tests/golden/plan_snapshots.json.gz from the UNMODIFIED reference:
PlannerInputs snapshots taken inside kvcsim.engine.Engine.step (the engine's
own plan_batch call, engine.py:616) together with the BatchPlan the reference
returned, so the device plan_batch (paper_2503_13773_b200.scheduler) can be
checked on the same inputs without the reference present.

    python oracle/make_plan_golden.py
"""
from __future__ import annotations

import copy
import gzip
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
REF = "/root/reference/pkg/src"
OUT = os.path.join(ROOT, "tests", "golden", "plan_snapshots.json.gz")

VIEW_FIELDS = ("req_id", "arrival_us", "kv_need", "generated", "estimated_total", "predicted_total", "allocated",
               "used", "slo_ttft_us", "slo_tbt_us", "remaining_ttft_us", "remaining_tbt_us", "ready",
               "prefill_done", "preemption_count", "is_guest", "tbt_blown")


def view_doc(v):
    d = {k: getattr(v, k) for k in VIEW_FIELDS}
    d["state"] = v.state.value
    return d


def pool_doc(pool):
    recs = []
    for o in pool.owners():
        recs.append({"id": o, "granted": pool.granted_of(o), "host": pool.host_of(o), "offset": pool.offset_of(o),
                     "guests": pool.guests_of(o), "reserved": pool.reserved_drawn_of(o), "used": pool.used_of(o)})
    return {"capacity": pool.capacity, "block_size": pool.block_size, "reserved_target": pool.reserved_target,
            "buffer_b": pool.buffer_b, "allow_stacking": pool.allow_stacking,
            "reserved_current": pool.reserved_blocks_current, "records": recs}


def plan_doc(plan):
    return {"members": [[m.req_id, m.tokens] for m in plan.members], "batch_tokens": plan.batch_tokens,
            "preempt": [[i, s.value] for i, s in plan.preempt],
            "actions": [[a.kind, a.req_id, a.tokens, a.blocks,
                         None if a.quote is None else [a.quote.host, a.quote.start_offset, a.quote.feasible_slack]]
                        for a in plan.actions],
            "claims": [list(c) for c in plan.claims], "deferred": list(plan.deferred), "overflow": plan.overflow}


def interesting(plan):
    return bool(plan.preempt or plan.claims or plan.deferred or
                any(a.kind in ("embed", "reserve") for a in plan.actions))


def main():
    sys.path.insert(0, REF)
    import kvcsim.engine as KE
    from dataclasses import asdict
    from oracle.make_golden import ref_build
    from tests.cases import case_params
    rnd = random.Random(0)
    snaps = []
    runs = [(s, None, False, False) for s in (0, 1, 2, 5, 13, 21)] + [(8, None, True, False), (27, None, True, False)] + \
        [(5, "vllm_block", False, False), (13, "sarathi_chunked", False, False), (6, "rlp", False, False),
         (2, "s3", False, False)] + \
        [(s, None, False, True) for s in (7, 9, 12)]  # invert_amortization=True (scheduler.py:233)
    for seed, pol, stack, inv in runs:
        p = case_params(seed)
        if pol:
            p["sched"] = {**p["sched"], "policy": pol}
        if inv:
            p["sched"] = {**p["sched"], "invert_amortization": True}
        p["allow_stacking"] = stack
        reqs, cfg = ref_build(p)
        got = []
        orig = KE.plan_batch

        def spy(inp, scfg):
            plan = orig(inp, scfg)
            n = len(inp.waiting) + len(inp.running)
            if n <= 400 and (interesting(plan) or rnd.random() < 0.01):
                got.append({
                    "run": f"seed{seed}-{pol or 'cacheopt'}{'-stack' if stack else ''}{'-inv' if inv else ''}",
                    "waiting": [view_doc(v) for v in inp.waiting], "running": [view_doc(v) for v in inp.running],
                    "pool": pool_doc(inp.pool), "t_i_max_us": inp.t_i_max_us,
                    "iter_cost": asdict(inp.iter_cost), "swap_model": asdict(inp.swap_model),
                    "recompute_model": asdict(inp.recompute_model),
                    "sched": {k: v for k, v in asdict(scfg).items() if k != "buckets"},
                    "buckets": asdict(scfg.buckets), "plan": plan_doc(plan)})
            return plan

        KE.plan_batch = spy
        try:
            eng = KE.Engine(copy.deepcopy(reqs), cfg)
            eng.run()
        finally:
            KE.plan_batch = orig
        # the rarer plan features first (reserve draws, deferrals, claims,
        # embeddings, preemptions), then random snapshots, 8 per run
        feats = (lambda d: any(a[0] == "reserve" for a in d["plan"]["actions"]), lambda d: d["plan"]["deferred"],
                 lambda d: d["plan"]["claims"], lambda d: any(a[0] == "embed" for a in d["plan"]["actions"]),
                 lambda d: d["plan"]["preempt"])
        take = []
        for f in feats:
            pool_f = [d for d in got if f(d) and d not in take]
            take += rnd.sample(pool_f, min(2, len(pool_f), 8 - len(take)))
        rest = [d for d in got if d not in take]
        take += rnd.sample(rest, min(len(rest), 8 - len(take)))
        print(f"seed {seed} {pol} stack={stack} inv={inv}: {len(got)} candidate snapshots, kept {len(take)}")
        snaps.extend(take)
    with open(OUT, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", mtime=0) as fh:
        fh.write(json.dumps(snaps).encode())
    print(f"{len(snaps)} snapshots -> {OUT}")


if __name__ == "__main__":
    main()
