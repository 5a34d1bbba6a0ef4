"""The reference's pure scheduling ops (scheduler.py:71-279) and victim
ordering (preemption.py:38-75) with their names and argument meaning.

The ops that make decisions -- classify_critical, fill_token_budget,
allocate_remaining, pair_release, proactive_include, order_victims -- run on
the GPU through the planner's own device code (csrc/sched_ops.cuh via
co_sched_op): the same criticality predicate, queue keys, block compaction,
rank sort, budget prefix, exact integer amortization and argmins k_plan uses
inside the engine step.  The closed-form demand helpers are host arithmetic,
as in the reference.  The engine never calls this module (its planner reads
the resident request pool); it exists so callers and the reference's own
tests can drive the device ops on snapshot views."""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass
from typing import Dict, Iterable, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .config import BucketConfig
from .core import Lifecycle

SOP_CLASSIFY, SOP_FILL_BUDGET, SOP_ALLOCATE_REMAINING, SOP_PAIR_RELEASE, SOP_ORDER_VICTIMS, \
    SOP_PROACTIVE_INCLUDE = range(6)
_DEVICE = 0


def set_device(device: int) -> None:
    """CUDA device the ops run on (default 0)."""
    global _DEVICE
    _DEVICE = int(device)


@dataclass(frozen=True)
class ReqView:
    """scheduler.py:71-96: the per-request snapshot handed to the planner."""
    req_id: int
    arrival_us: int
    state: Lifecycle
    kv_need: int
    generated: int
    estimated_total: int
    predicted_total: int
    allocated: int
    used: int
    slo_ttft_us: int
    slo_tbt_us: int
    remaining_ttft_us: Optional[int]
    remaining_tbt_us: Optional[int]
    ready: bool = True
    prefill_done: int = 0
    preemption_count: int = 0
    is_guest: bool = False
    tbt_blown: bool = False


def est_remaining(v: ReqView) -> int:
    return max(0, v.estimated_total - v.generated)


def target_alloc(v: ReqView) -> int:
    return max(v.used, v.kv_need) + est_remaining(v)


def rt_us(v: ReqView) -> int:
    if v.remaining_ttft_us is not None:
        return v.remaining_ttft_us
    if v.remaining_tbt_us is None:
        raise AssertionError("a view needs remaining_ttft_us or remaining_tbt_us")
    return v.remaining_tbt_us


def is_returned(v: ReqView) -> bool:
    return v.state is Lifecycle.RUNNING and v.allocated < v.used + 1


@dataclass
class CriticalSets:
    n_w: List[ReqView]
    n_r: List[ReqView]
    n_w_prime: List[ReqView]
    n_r_prime: List[ReqView]


@dataclass(frozen=True)
class AllocDemand:
    req_id: int
    m_tokens: int
    rt_us: int
    prompt_len: int


@dataclass(frozen=True)
class PairCandidate:
    req_id: int
    est_remaining_iters: int
    release_gain: int


@dataclass(frozen=True)
class VictimInfo:
    req_id: int
    slo_tbt_us: int
    remaining_tokens: int
    occupancy_tokens: int


def _ranks(ids: Sequence[int]) -> np.ndarray:
    order = np.argsort(np.asarray(ids, dtype=np.int64), kind="stable")
    r = np.empty(len(ids), dtype=np.int64)
    r[order] = np.arange(len(ids))
    return r


def _run(op: int, rows: np.ndarray, params: Sequence[int]) -> np.ndarray:
    lib = N.load()
    n = len(rows)
    rows = np.ascontiguousarray(rows, dtype=np.int64).reshape(n, 8) if n else np.zeros((0, 8), dtype=np.int64)
    prm = np.zeros(16, dtype=np.int64)
    prm[:len(params)] = params
    out = np.zeros(2 * max(n, 1) + 8, dtype=np.int64)
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    N.check(lib.co_sched_op(op, n, p(rows), p(prm), p(out), _DEVICE), "co_sched_op")
    return out


# -- criticality (scheduler.py:129-163) -----------------------------------------

def classify_critical(waiting: Sequence[ReqView], running: Sequence[ReqView], t_i_max_us: int,
                      epsilon_us: int) -> CriticalSets:
    views = list(waiting) + list(running)
    rows = np.zeros((len(views), 8), dtype=np.int64)
    rows[:, 0] = _ranks([v.req_id for v in views])
    for k, v in enumerate(views):
        run = k >= len(waiting)
        rows[k, 1] = int(run)
        if run:
            ret = is_returned(v)
            rows[k, 3] = int(ret)
            if ret:
                if v.remaining_tbt_us is None:
                    raise AssertionError("a returned running view needs remaining_tbt_us")
                rows[k, 2] = v.remaining_tbt_us
        else:
            rows[k, 2] = rt_us(v)
        rows[k, 4] = v.arrival_us
    out = _run(SOP_CLASSIFY, rows, [t_i_max_us, epsilon_us])
    cnt = out[:4].tolist()
    lists, base = [], 4
    for c in cnt:
        lists.append([views[int(x)] for x in out[base:base + c]])
        base += c
    return CriticalSets(n_w=lists[0], n_r=lists[1], n_w_prime=lists[2], n_r_prime=lists[3])


# -- demand arithmetic (scheduler.py:166-179) ------------------------------------

def basic_demand(sets: CriticalSets, small_block_b: int) -> int:
    need = sum(max(0, v.kv_need + small_block_b - v.allocated) for v in sets.n_w)
    return need + small_block_b * len(sets.n_r)


def ensure_capacity(pool_free: int, d_kvc: int) -> int:
    return max(0, d_kvc - pool_free)


# -- token budget (scheduler.py:182-200) -----------------------------------------

def fill_token_budget(sets: CriticalSets, waiting_ordered: Sequence[ReqView], token_budget: int,
                      consumed_tokens: int) -> Tuple[List[ReqView], bool]:
    q = list(waiting_ordered)
    rows = np.zeros((len(q), 8), dtype=np.int64)
    for k, v in enumerate(q):
        rows[k, 0] = v.kv_need - v.prefill_done
    out = _run(SOP_FILL_BUDGET, rows, [token_budget, consumed_tokens])
    return q[:int(out[0])], bool(out[1])


# -- remaining-KVC amortization (scheduler.py:211-243) ---------------------------

def allocate_remaining(demands: Sequence[AllocDemand], a_prime: int, invert: bool = False) -> Dict[int, int]:
    if a_prime < 0:
        raise ValueError("a_prime must be >= 0")
    ds = list(demands)
    if not ds:
        return {}
    rows = np.zeros((len(ds), 8), dtype=np.int64)
    rows[:, 0] = _ranks([d.req_id for d in ds])
    for k, d in enumerate(ds):
        rows[k, 1:4] = (d.m_tokens, d.rt_us, d.prompt_len)
    out = _run(SOP_ALLOCATE_REMAINING, rows, [a_prime, int(bool(invert))])
    return {d.req_id: int(out[k]) for k, d in enumerate(ds) if d.m_tokens > 0}


# -- pair release and proactive inclusion (scheduler.py:253-279) -----------------

def pair_release(residual_tokens: int, runway_iters: int, candidates: Sequence[PairCandidate]) -> Optional[int]:
    cs = list(candidates)
    if not cs:
        return None
    rows = np.zeros((len(cs), 8), dtype=np.int64)
    rows[:, 0] = _ranks([c.req_id for c in cs])
    for k, c in enumerate(cs):
        rows[k, 1:3] = (c.est_remaining_iters, c.release_gain)
    k = int(_run(SOP_PAIR_RELEASE, rows, [residual_tokens, runway_iters])[0])
    return None if k < 0 else cs[k].req_id


def proactive_include(running: Sequence[ReqView], m: int) -> List[ReqView]:
    rs = list(running)
    rows = np.zeros((len(rs), 8), dtype=np.int64)
    if rs:
        rows[:, 0] = _ranks([v.req_id for v in rs])
    for k, v in enumerate(rs):
        rows[k, 1:5] = (int(is_returned(v)), v.allocated, target_alloc(v), est_remaining(v))
    out = _run(SOP_PROACTIVE_INCLUDE, rows, [m])
    return [rs[int(x)] for x in out[1:1 + int(out[0])]]


# -- baseline grant arithmetic (scheduler.py:282-288) ----------------------------

def s3_demand(predicted: int, bucket_tokens: int, preempt_count: int) -> int:
    buckets = max(1, math.ceil(max(1, predicted) / bucket_tokens))
    return buckets * bucket_tokens * (2 ** preempt_count)


def rlp_demand(predicted_remaining: int, padding: int) -> int:
    return max(1, predicted_remaining) + padding


# -- victim ordering (preemption.py:38-75) ----------------------------------------

def victim_key(slo_tbt_us: int, remaining_tokens: int, occupancy_tokens: int, req_id: int,
               cfg: BucketConfig) -> Tuple[int, int, int, int]:
    slo_b = sum(1 for e in cfg.slo_edges_us if slo_tbt_us >= e)
    return (-slo_b, -(max(0, remaining_tokens) // cfg.token_step), occupancy_tokens, req_id)


def order_victims(candidates: Iterable[VictimInfo], cfg: BucketConfig) -> List[VictimInfo]:
    vs = list(candidates)
    if not vs:
        return []
    edges = list(cfg.slo_edges_us)
    if len(edges) > 6:
        raise ValueError("at most 6 SLO bucket edges on the device")
    rows = np.zeros((len(vs), 8), dtype=np.int64)
    rows[:, 0] = _ranks([v.req_id for v in vs])
    for k, v in enumerate(vs):
        rows[k, 1:4] = (v.slo_tbt_us, v.remaining_tokens, v.occupancy_tokens)
    out = _run(SOP_ORDER_VICTIMS, rows, [cfg.token_step, len(edges)] + edges)
    return [vs[int(x)] for x in out[:len(vs)]]


# -- the planner operator on a snapshot (scheduler.py:295-335, 939-950) -----------

@dataclass
class PlanAction:
    kind: str
    req_id: int
    tokens: int = 0
    blocks: int = 0
    quote: Optional[object] = None  # kvc.EmbedQuote for "embed"


@dataclass(frozen=True)
class PlanMember:
    req_id: int
    tokens: int


@dataclass
class BatchPlan:
    members: List[PlanMember]
    batch_tokens: int = 0
    preempt: List[Tuple[int, object]] = None
    actions: List[PlanAction] = None
    claims: List[Tuple[int, int]] = None
    deferred: List[int] = None
    overflow: bool = False


@dataclass
class PlannerInputs:
    waiting: List[ReqView]
    running: List[ReqView]
    pool: object          # kvc.BlockPool (device) or the reference's BlockPool: queried read-only
    t_i_max_us: int
    iter_cost: object     # config.IterationCost
    swap_model: object    # config.SwapModel
    recompute_model: object


_ACT = ("allocate", "grow", "reserve", "embed")
_NOW = 1 << 40  # snapshot clock: every signed slack maps to positive device times


def plan_batch(inp: PlannerInputs, cfg, device: Optional[int] = None) -> BatchPlan:
    """scheduler.py:939-950 on the device: the snapshot's views and pool
    records are loaded into an engine's request pool and ONE pass of the
    device planner (k_classify + k_serial's plan_body, every policy of
    POLICIES) produces the plan.  The engine gives its planner the live set
    in arrival order (engine.py:321-323); the views are taken in that order."""
    from .config import EngineConfig, TruthCosts
    from .core import Request, Strategy
    from .engine import Engine
    from .kvc import EmbedQuote
    pool = inp.pool
    if pool.block_size != cfg.small_block_b:
        raise ValueError("the pool's block size must be the scheduler's small_block_b (engine.py:236)")
    views = sorted(list(inp.waiting) + list(inp.running), key=lambda v: (v.arrival_us, v.req_id))
    n = len(views)
    ids = [v.req_id for v in views]
    if len(set(ids)) != n:
        raise ValueError("duplicate request ids in the snapshot")
    idx = {r: k for k, r in enumerate(ids)}
    owners = list(pool.owners())
    for o in owners:
        if o not in idx:
            raise ValueError(f"pool record {o} has no view in the snapshot")
    reqs = []
    cols = np.zeros((n, 20), dtype=np.int64)
    code = {Lifecycle.WAITING: 1, Lifecycle.RUNNING: 2, Lifecycle.PREEMPTED: 3}
    for k, v in enumerate(views):
        if v.state not in code:
            raise ValueError(f"view {v.req_id}: state {v.state} is not live")
        if v.remaining_ttft_us is not None:       # no first token: rt = slo_ttft - (now - arrival)
            slo_ttft, first, last = v.remaining_ttft_us + _NOW - v.arrival_us, -1, -1
        else:
            slo_ttft, first = v.slo_ttft_us, 0
            last = v.remaining_tbt_us - v.slo_tbt_us + _NOW  # rt = slo_tbt - (now - last_token)
        out_len = max(1, v.used + 2 - max(1, v.kv_need), v.generated + 1, v.predicted_total, v.estimated_total)
        reqs.append(Request(id=v.req_id, arrival_us=v.arrival_us, prompt_len=max(1, v.kv_need),
                            true_output_len=out_len, slo_ttft_us=slo_ttft, slo_tbt_us=v.slo_tbt_us))
        cols[k, :12] = (code[v.state], v.generated, v.used, v.kv_need, v.prefill_done, v.preemption_count,
                        v.predicted_total, v.estimated_total, first, last,
                        v.slo_tbt_us + 1 if v.tbt_blown else 0, _NOW if v.ready else _NOW + 1)
    cols[:, 14] = -1
    cols[:, 17] = -1
    cols[:, 18] = -1
    fp = lambda t: -(-t // pool.block_size) * pool.block_size  # noqa: E731
    fp_sum = g_sum = u_sum = 0
    for seq, o in enumerate(owners, start=1):  # owners() is the records' creation order
        k = idx[o]
        g = pool.granted_of(o)
        h = pool.host_of(o)
        cols[k, 12:17] = (1, g, -1 if h is None else idx[h], pool.offset_of(o), pool.reserved_drawn_of(o))
        cols[k, 19] = seq
        gl = [idx[x] for x in pool.guests_of(o)]
        if gl:
            cols[k, 17] = gl[0]
            for a, b in zip(gl, gl[1:]):
                cols[a, 18] = b
        g_sum += g
        u_sum += pool.used_of(o)
        if h is None:
            fp_sum += fp(g)
        if pool.used_of(o) != views[k].used:
            raise ValueError(f"request {o}: pool used {pool.used_of(o)} != view used {views[k].used}")
    ecfg = EngineConfig(capacity_tokens=pool.capacity, reserved_blocks=pool.reserved_target,
                        allow_stacking=bool(getattr(pool, "allow_stacking", False)), sched=cfg,
                        iter_cost=inp.iter_cost, truth=TruthCosts(inp.swap_model, inp.recompute_model),
                        record_events=False)
    eng = Engine(reqs, ecfg, device=_DEVICE if device is None else device)
    try:
        if eng._rid != ids:
            raise AssertionError("engine order differs from the snapshot order")
        scal = np.array([_NOW, inp.t_i_max_us, pool.reserved_blocks_current, fp_sum, g_sum, u_sum, len(owners), n],
                        dtype=np.int64)
        hdr = np.zeros(8, dtype=np.int64)
        cap = 12 * n + 64
        lists = np.zeros(cap, dtype=np.int32)
        p64 = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
        N.check(eng._lib.co_plan_snapshot(eng._h, p64(np.ascontiguousarray(cols)), p64(scal), p64(hdr),
                                          lists.ctypes.data_as(C.POINTER(C.c_int32)), cap), "co_plan_snapshot")
    finally:
        eng.close()
    nm, na, npre, ncl, nd = (int(x) for x in hdr[:5])
    it = iter(np.split(lists, np.cumsum([nm, nm, na, na, na, na, na, na, npre, npre, ncl, ncl, nd]))[:13])
    mi, mt, ak, ai, at, anb, ah, ast, pi, ps, cw, cp, di = (a.tolist() for a in it)
    plan = BatchPlan(members=[PlanMember(ids[i], t) for i, t in zip(mi, mt)], batch_tokens=int(hdr[6]),
                     preempt=[(ids[i], Strategy.SWAP if s == 0 else Strategy.RECOMPUTE) for i, s in zip(pi, ps)],
                     actions=[], claims=[(ids[w], ids[p]) for w, p in zip(cw, cp)], deferred=[ids[i] for i in di],
                     overflow=bool(hdr[5]))
    for kind, i, tok, nb, h, start in zip(ak, ai, at, anb, ah, ast):
        quote = None
        if _ACT[kind] == "embed":
            out = tok - views[i].kv_need  # need = kv_need + out (scheduler.py:438-441)
            quote = EmbedQuote(host=ids[h], start_offset=start, feasible_slack=start - views[h].used - out)
        plan.actions.append(PlanAction(_ACT[kind], ids[i], tokens=tok, blocks=nb, quote=quote))
    return plan
