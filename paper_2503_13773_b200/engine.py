"""Drop-in engine: the reference's ``Engine`` surface (engine.py:222-672)
backed by the device engine in libcacheopt.so.

``Engine(requests, cfg)`` uploads the trace once, ``step()`` runs one device
scheduling round, ``run()`` runs the whole trace as CUDA-graph launches and
returns the same ``MetricsReport``.  ``events``, ``runtimes``, ``requests`` and
``pool`` are host views materialised from device readbacks on access.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import json
import math
from dataclasses import dataclass
from typing import Dict, Iterator, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N
from .build import hostlog_path
from .config import DEVICE_POLICIES, EngineConfig
from .core import (STATE_FROM_CODE, STRATEGY_FROM_CODE, US_PER_S, Direction, LengthEstimate,
                   Lifecycle, Request, RequestRuntime, Strategy)
from .devrng import predictor_draws_device
from .hostprep import (bin_of, charge_luts, iteration_us, run_confidence, run_padding,
                       sweet_spot)

STRATEGY_CODE = {Strategy.SWAP: 0, Strategy.RECOMPUTE: 1}


_hostlog = None


def _load_hostlog():
    global _hostlog
    if _hostlog is not None:
        return _hostlog
    import importlib.machinery
    import importlib.util
    path = hostlog_path()
    if not path.exists():
        raise N.NativeError(f"{path.name} not built: run __graft_entry__.build()")
    loader = importlib.machinery.ExtensionFileLoader("paper_2503_13773_b200._hostlog", str(path))
    spec = importlib.util.spec_from_file_location("paper_2503_13773_b200._hostlog", str(path), loader=loader)
    mod = importlib.util.module_from_spec(spec)
    loader.exec_module(mod)
    _hostlog = mod
    return mod


_STRATEGY_NAMES = tuple(STRATEGY_FROM_CODE[k].value for k in range(2))
_CAUSE_NAMES = tuple(N.CAUSES)

CAUSE_CODE = {"plan": 0, "squeeze": 1, "collision": 2}


@dataclass
class MetricsReport:
    policy: str
    seed: int
    num_requests: int
    completed: int
    makespan_us: int
    ttft_us: Dict[str, float]
    tbt_us: Dict[str, float]
    ttft_attainment: float
    tbt_attainment: float
    normalized_us_per_token: Dict[str, float]
    preemption_total: int
    preempted_requests: int
    preemption_time_us: Dict[str, float]
    throughput_rps: float
    throughput_tps: float
    kvc_utilization_mean: float
    kvc_fragmentation_mean: float
    waiting_us_mean: float
    execution_us_mean: float
    preemption_us_mean: float

    def to_dict(self) -> dict:
        return dataclasses.asdict(self)


def _pct(values) -> Dict[str, float]:
    if len(values) == 0:
        return {"p50": 0.0, "p90": 0.0, "p99": 0.0, "max": 0.0, "mean": 0.0}
    a = np.asarray(values, dtype=float)
    return {"p50": float(np.percentile(a, 50)), "p90": float(np.percentile(a, 90)),
            "p99": float(np.percentile(a, 99)), "max": float(a.max()), "mean": float(a.mean())}


def pct_from_order_stats(count: int, os7: Sequence[float], total) -> Dict[str, float]:
    """_pct's dict from the order statistics co_metrics selects: np.percentile
    'linear' (virtual index (n-1)q, _lerp's two-sided form) at q = .5/.9/.99
    between os7[2j] and os7[2j+1], max = os7[6], mean = sum / n (``total`` is
    the exact integer sum, or the numpy-pairwise float sum)."""
    if count == 0:
        return {"p50": 0.0, "p90": 0.0, "p99": 0.0, "max": 0.0, "mean": 0.0}
    out = {}
    for j, (name, q) in enumerate((("p50", 50 / 100), ("p90", 90 / 100), ("p99", 99 / 100))):
        a, b = float(os7[2 * j]), float(os7[2 * j + 1])
        v = (count - 1) * q
        g = v - math.floor(v) if v < count - 1 else 0.0
        d = b - a
        out[name] = b - d * (1 - g) if g >= 0.5 else a + d * g
    out["max"] = float(os7[6])
    out["mean"] = float(total) / count
    return out


def order_stat_ranks(count: int) -> List[int]:
    """The ranks co_metrics selects (host restatement, for tests)."""
    r = []
    for q in (50 / 100, 90 / 100, 99 / 100):
        v = (count - 1) * q
        lo = count - 1 if v >= count - 1 else math.floor(v)
        r += [lo, count - 1 if v >= count - 1 else lo + 1]
    return r + [count - 1]


def compute_metrics(*, requests: Dict[int, Request], runtimes: Dict[int, RequestRuntime], policy: str,
                    seed: int, makespan_us: int, capacity_tokens: int,
                    samples: Sequence[Tuple[int, int]]) -> MetricsReport:
    """Outcome aggregation with the reference's definitions (engine.py:132-211):
    latency percentiles over completed requests, attainment over all of
    them, utilization/fragmentation from per-iteration (footprint, used)."""
    n = len(requests)
    ttfts, gaps_all, norm, waits, execs, pdec = [], [], [], [], [], []
    ok_ttft = ok_tbt = done = 0
    for rid, req in requests.items():
        rt = runtimes[rid]
        tt = rt.token_times_us
        gaps = [b - a for a, b in zip(tt, tt[1:])]
        if rt.first_token_at_us is not None and rt.first_token_at_us - req.arrival_us <= req.slo_ttft_us:
            ok_ttft += 1
        if req.state is not Lifecycle.COMPLETED:
            continue
        done += 1
        if all(g <= req.slo_tbt_us for g in gaps):
            ok_tbt += 1
        ttfts.append(rt.first_token_at_us - req.arrival_us)
        gaps_all.extend(gaps)
        norm.append((rt.completion_us - req.arrival_us) / req.true_output_len)
        waits.append(rt.first_start_us - req.arrival_us)
        pdec.append(rt.preemption_time_us)
        execs.append(rt.completion_us - rt.first_start_us - rt.preemption_time_us)
    hit = [rt for rt in runtimes.values() if rt.preemption_count > 0]
    span_s = makespan_us / US_PER_S if makespan_us > 0 else 0.0
    gen_total = sum(rt.generated for rt in runtimes.values())
    if len(samples):
        util = float(np.mean([fp / capacity_tokens for fp, _ in samples]))
        frag = float(np.mean([(fp - u) / capacity_tokens for fp, u in samples]))
    else:
        util = frag = 0.0

    def mean(xs):
        return float(np.mean(xs)) if xs else 0.0

    return MetricsReport(
        policy=policy, seed=seed, num_requests=n, completed=done, makespan_us=makespan_us,
        ttft_us=_pct(ttfts), tbt_us=_pct(gaps_all),
        ttft_attainment=ok_ttft / n if n else 0.0, tbt_attainment=ok_tbt / n if n else 0.0,
        normalized_us_per_token=_pct(norm),
        preemption_total=sum(rt.preemption_count for rt in runtimes.values()),
        preempted_requests=len(hit), preemption_time_us=_pct([rt.preemption_time_us for rt in hit]),
        throughput_rps=done / span_s if span_s else 0.0,
        throughput_tps=gen_total / span_s if span_s else 0.0,
        kvc_utilization_mean=util, kvc_fragmentation_mean=frag,
        waiting_us_mean=mean(waits), execution_us_mean=mean(execs), preemption_us_mean=mean(pdec),
    )


def calibrate_slo_baselines(requests: Sequence[Request], cfg: EngineConfig, device: int = -1
                            ) -> Tuple[int, int]:
    """engine.py:675-699: median per-chunk TTFT and median token gap of a
    vllm_block run (which ignores SLOs) -- the simulation runs on the device
    (the baseline planner of csrc/planner.cuh), the two medians on the host."""
    cal_cfg = dataclasses.replace(cfg, sched=dataclasses.replace(cfg.sched, policy="vllm_block"),
                                  record_events=False)
    eng = Engine(list(requests), cal_cfg, device=device)
    try:
        eng.run_steps(0)
        st = eng._field("STATE")
        ft = eng._field("FIRST_TOKEN")
        offs = np.empty(eng._n + 1, dtype=np.int64)
        times = np.empty(max(1, int(eng._tok_total())), dtype=np.int64)
        N.check(eng._lib.co_read_token_times(eng._h, _ptr(offs, C.c_int64), _ptr(times, C.c_int64)),
                "co_read_token_times")
        gen = eng._field("GENERATED")
    finally:
        eng.close()
    chunk = cfg.sched.token_budget
    by_id = {r.id: r for r in requests}
    ttfts, gaps = [], []
    for r in requests:  # the reference iterates eng.requests (caller order)
        k = eng._idx_of[r.id]
        if STATE_FROM_CODE[int(st[k])] is not Lifecycle.COMPLETED:
            continue
        factor = max(1, -(-by_id[r.id].prompt_len // chunk))
        ttfts.append((int(ft[k]) - r.arrival_us) / factor)
        t = times[offs[k]:offs[k] + int(gen[k])]
        gaps.extend(np.diff(t).tolist())
    if not ttfts or not gaps:
        raise ValueError("calibration run completed no requests")
    return int(np.median(ttfts)), int(np.median(gaps))


def write_events_jsonl(events: Sequence[dict], path: str) -> None:
    """One sorted-key compact JSON object per line (engine.py:214-219)."""
    with open(path, "w") as fh:
        for ev in events:
            fh.write(json.dumps(ev, sort_keys=True, separators=(",", ":")))
            fh.write("\n")


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(C.POINTER(ct))


class PoolView:
    """Read-only view of the device KV pool with the BlockPool query API
    (kvc.py:86-140)."""

    def __init__(self, eng: "Engine"):
        self._e = eng

    def _f(self, name):
        return self._e._field(name)

    @property
    def capacity(self) -> int:
        return self._e.cfg.capacity_tokens

    @property
    def block_size(self) -> int:
        return self._e.cfg.sched.small_block_b

    @property
    def buffer_b(self) -> int:
        return self._e.cfg.sched.buffer_b

    @property
    def reserved_target(self) -> int:
        return self._e.cfg.reserved_blocks

    @property
    def reserved_blocks_current(self) -> int:
        return int(self._e._scalars().reserved_blocks_current)

    @property
    def free_tokens(self) -> int:
        s = self._e._scalars()
        return self.capacity - s.reserved_blocks_current * self.block_size - s.footprint_tokens

    @property
    def footprint_tokens(self) -> int:
        return int(self._e._scalars().footprint_tokens)

    @property
    def granted_tokens(self) -> int:
        return int(self._e._scalars().granted_tokens)

    @property
    def used_tokens(self) -> int:
        return int(self._e._scalars().used_tokens)

    def _idx(self, rid: int) -> int:
        k = self._e._idx_of.get(rid)
        if k is None or not self._f("HOLDS")[k]:
            raise ValueError(f"no allocation for request {rid}")
        return k

    def holds(self, rid: int) -> bool:
        k = self._e._idx_of.get(rid)
        return k is not None and bool(self._f("HOLDS")[k])

    def granted_of(self, rid: int) -> int:
        return int(self._f("GRANTED")[self._idx(rid)])

    def used_of(self, rid: int) -> int:
        return int(self._f("USED")[self._idx(rid)])

    def host_of(self, rid: int) -> Optional[int]:
        h = int(self._f("HOST")[self._idx(rid)])
        return None if h < 0 else self._e._rid[h]

    def offset_of(self, rid: int) -> int:
        k = self._idx(rid)
        return int(self._f("EMBED_OFFSET")[k]) if self._f("HOST")[k] >= 0 else 0

    def reserved_drawn_of(self, rid: int) -> int:
        return int(self._f("RESERVED_DRAWN")[self._idx(rid)])

    def guests_of(self, rid: int) -> List[int]:
        """kvc.py:124-125: the host's guests in embed order (= their records'
        creation order: a guest record is created by the embed)."""
        k = self._idx(rid)
        host = self._f("HOST")
        holds = self._f("HOLDS")
        seq = self._f("RECORD_SEQ")
        g = np.nonzero((host == k) & (holds == 1))[0]
        return [self._e._rid[x] for x in g[np.argsort(seq[g], kind="stable")]]

    def owners(self) -> List[int]:
        holds = self._f("HOLDS")
        seq = self._f("RECORD_SEQ")
        idx = np.nonzero(holds)[0]
        return [self._e._rid[k] for k in idx[np.argsort(seq[idx], kind="stable")]]


class _Runtimes(dict):
    pass


class Engine:
    """Device-backed drop-in for the reference Engine (policy ``cacheopt``)."""

    def __init__(self, requests: Sequence[Request], cfg: EngineConfig, device: int = -1,
                 steps_per_launch: int = 32, kv: Optional["KVLayout"] = None):
        ids = [r.id for r in requests]
        if len(set(ids)) != len(ids):
            raise ValueError("request ids must be unique")
        if cfg.sched.policy not in DEVICE_POLICIES:
            raise ValueError(f"policy {cfg.sched.policy!r} has no device implementation "
                             f"(device policies: {DEVICE_POLICIES})")
        self.cfg = cfg
        # the caller's Request objects, kept current like the reference's
        # in-step transitions (core.py:113-130): refreshed lazily on access
        self._requests: Dict[int, Request] = {r.id: r for r in requests}
        self._req_stale = False
        self._input_order = ids
        self.steps_per_launch = steps_per_launch
        lib = N.load()
        n = len(requests)
        req_id = np.array(ids, dtype=np.int64)
        arr = np.array([r.arrival_us for r in requests], dtype=np.int64)
        prompt = np.array([r.prompt_len for r in requests], dtype=np.int32)
        tout = np.array([r.true_output_len for r in requests], dtype=np.int32)
        ttft = np.array([r.slo_ttft_us for r in requests], dtype=np.int64)
        tbt = np.array([r.slo_tbt_us for r in requests], dtype=np.int64)
        order = np.lexsort((req_id, arr)) if n else np.zeros(0, dtype=np.int64)
        self._rid = [int(x) for x in req_id[order]]
        self._idx_of = {r: k for k, r in enumerate(self._rid)}
        arr_sorted = arr[order]
        self.confidence = run_confidence(cfg, arr_sorted)
        self.padding = run_padding(cfg, self.confidence)
        # estimation.py:76-99 noise, drawn on the GPU from default_rng([seed, 3])
        err_d, flip_d = predictor_draws_device(cfg.predictor, cfg.seed, n, device)
        err, flip = err_d.cpu().numpy(), flip_d.cpu().numpy()
        s_max = int((prompt.astype(np.int64) + tout).max()) if n else 1
        luts = charge_luts(cfg, max(s_max, 1))
        self._keep = [req_id, arr, prompt, tout, ttft, tbt, err, flip, *luts]
        tout_s = tout[order].astype(np.int64)
        pred_s = np.maximum(1, tout_s - err)
        self._under = (tout_s >= pred_s) ^ (flip.astype(bool))  # estimation.py:96-98
        sc = cfg.sched
        edges = list(sc.buckets.slo_edges_us)
        if len(edges) > N.MAX_SLO_EDGES:
            raise ValueError("at most 8 SLO bucket edges are supported")
        c = N.CoConfig()
        c.capacity_tokens = cfg.capacity_tokens
        c.reserved_blocks = cfg.reserved_blocks
        c.allow_stacking = int(cfg.allow_stacking)
        c.invert_amortization = int(sc.invert_amortization)  # scheduler.py:43, :233
        c.block_size = sc.small_block_b
        c.buffer_b = sc.buffer_b
        c.token_budget = sc.token_budget
        c.preallocate_m = sc.preallocate_m
        c.decode_runway_iters = sc.decode_runway_iters
        c.victim_rule_fcfs = 1 if sc.victim_rule == "fcfs" else 0
        c.epsilon_us = sc.epsilon_us
        c.n_slo_edges = len(edges)
        c.token_step = sc.buckets.token_step
        for k, e in enumerate(edges):
            c.slo_edges_us[k] = int(e)
        c.iter_base_ms = float(cfg.iter_cost.base_ms)
        c.iter_per_token_ms = float(cfg.iter_cost.per_token_ms)
        c.horizon_factor = cfg.horizon_factor
        c.validate_every = cfg.validate_every
        c.record_events = int(cfg.record_events)
        c.padding = self.padding
        c.s_star = sweet_spot(cfg.truth.swap_true, cfg.truth.recompute_true)
        c.t_i_init_us = iteration_us(cfg, sc.token_budget)
        c.policy = N.POLICY_CODE[sc.policy]
        c.vllm_block_tokens, c.s3_bucket_tokens, c.rlp_padding = sc.vllm_block_tokens, sc.s3_bucket_tokens, sc.rlp_padding
        self.kv = kv
        if kv is not None:
            c.kv_layers, c.kv_heads, c.q_heads, c.head_dim = kv.layers, kv.kv_heads, kv.q_heads, kv.head_dim
            c.host_swap_pages = kv.host_swap_pages
            c.decode = int(kv.decode)
            c.decode_split = kv.decode_split
        t = N.CoTrace()
        t.n = n
        t.req_id = _ptr(req_id, C.c_int64)
        t.arrival_us = _ptr(arr, C.c_int64)
        t.prompt_len = _ptr(prompt, C.c_int32)
        t.true_output_len = _ptr(tout, C.c_int32)
        t.slo_ttft_us = _ptr(ttft, C.c_int64)
        t.slo_tbt_us = _ptr(tbt, C.c_int64)
        t.err_draw = _ptr(err, C.c_int32)
        t.flip_draw = _ptr(flip, C.c_uint8)
        lu = N.CoLuts()
        lu.s_max = max(s_max, 1)
        lu.swap_half_us, lu.recompute_us, lu.survive_swap_us, lu.survive_rec_us = (
            _ptr(x, C.c_int64) for x in luts)
        h = C.c_void_p()
        N.check(lib.co_create(C.byref(c), C.byref(t), C.byref(lu), device, C.byref(h)), "co_create")
        self._lib = lib
        self._h = h
        self._n = n
        self._events: List[dict] = []
        self._samples: List[Tuple[int, int]] = []
        self._cache: Dict[str, np.ndarray] = {}
        self._sc = None
        self.report: Optional[MetricsReport] = None
        self.pool = PoolView(self)
        self._resbuf = None
        self._evbuf = self._membuf = self._sbuf = None
        self._drain_args = None
        self._log_clean = False
        self._step_args = {}
        self._rid_np = np.array(self._rid, dtype=np.int64)
        self._cnt = (C.c_int64 * 3)()

    # -- lifecycle -----------------------------------------------------------

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.co_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _dirty(self) -> None:
        self._cache.clear()
        self._sc = None
        self._req_stale = True
        self._log_clean = False

    def _scalars(self) -> N.CoScalars:
        if self._sc is None:
            s = N.CoScalars()
            N.check(self._lib.co_get_scalars(self._h, C.byref(s)), "co_get_scalars")
            self._sc = s
        return self._sc

    def _field(self, name: str) -> np.ndarray:
        a = self._cache.get(name)
        if a is None:
            a = np.empty(self._n, dtype=np.int64)
            N.check(self._lib.co_read_field(self._h, N.FIELD[name], _ptr(a, C.c_int64)), "co_read_field")
            self._cache[name] = a
        return a

    # -- the reference surface ----------------------------------------------

    @property
    def now_us(self) -> int:
        return int(self._scalars().now_us)

    def step(self) -> bool:
        r = C.c_int32()
        self._dirty()
        N.check(self._lib.co_step(self._h, C.byref(r)), "co_step")
        return bool(r.value)

    def prepare_step(self) -> None:
        """Instantiate the per-step graph and result buffer now (no step runs),
        so the first step()/step_result() after this is not a capture."""
        N.check(self._lib.co_prepare_step(self._h), "co_prepare_step")

    def step_result(self, drain: bool = True):
        """step() plus this iteration's result in one device round trip:
        (step()'s bool, int64 array [m, 2] of (req_id, tokens) that ran, end_us).
        With `drain` (default) the step's event log and utilization sample
        come back in the same library call (co_step_packed -> co_step_result_log)
        into the host lists, so `events` then has nothing left to fetch."""
        drain = bool(drain and self.cfg.record_events)
        if self._resbuf is None:
            self._resbuf = np.empty(2 * (3 * self._n + 64), dtype=np.int64)  # (req_id, tokens) pairs
            self._sr_out = (C.c_int32(), C.c_int64(), C.c_int64())
        if drain and self._evbuf is None:
            self._drain()  # sizes the host log buffers once
        sa = self._step_args.get(drain)
        if sa is None:
            r, n, end = self._sr_out
            a = N.CoStepArgs(eng=self._h.value, result=C.addressof(r), members=None,
                             max_members=len(self._resbuf) // 2, n_members=C.addressof(n),
                             ids=self._rid_np.ctypes.data, members_ids=self._resbuf.ctypes.data,
                             iter_end_us=C.addressof(end), drain=int(drain))
            if drain:
                a.events, a.max_events = self._ev_addr, len(self._evbuf)
                a.log_members, a.max_log_members = self._mem_addr, len(self._membuf) // 2
                a.samples, a.max_samples = C.addressof(self._sbuf), len(self._sbuf) // 2
                a.counts = C.addressof(self._cnt)
            sa = self._step_args[drain] = (a, C.addressof(a))
        r, n, end = self._sr_out
        self._cache.clear()
        self._sc = None
        self._req_stale = True
        self._log_clean = False
        rc = self._lib.co_step_packed(sa[1])
        if drain:
            if rc == N.CO_EAGAIN:  # the step ran; its log needs larger buffers
                self._drain()
            elif rc:
                N.check(rc, "co_step_packed")
            else:
                self._take_log()
            self._log_clean = True
        elif rc:
            N.check(rc, "co_step_packed")
        k = n.value
        return bool(r.value), self._resbuf[:2 * k].reshape(k, 2).copy(), int(end.value)

    def run_steps(self, max_steps: int = 0, steps_per_launch: Optional[int] = None) -> int:
        """Device loop with the run() progress guard; returns step() calls."""
        k = steps_per_launch or self.steps_per_launch
        done = C.c_int64()
        self._dirty()
        N.check(self._lib.co_run(self._h, max_steps, k, C.byref(done)), "co_run")
        return int(done.value)

    def run(self) -> MetricsReport:
        """engine.py:643-672: run to completion, then the metrics, aggregated on
        the device (report_device); report_host() is the host restatement."""
        self.run_steps(0)
        self.report = self.report_device()
        return self.report

    def report_host(self) -> MetricsReport:
        """compute_metrics over host views of every request (engine.py:132-211)."""
        s = self._scalars()
        makespan = max(0, int(s.now_us) - int(s.first_arrival_us))
        return compute_metrics(
            requests=self.requests_view(), runtimes=self.runtimes, policy=self.cfg.sched.policy,
            seed=self.cfg.seed, makespan_us=makespan, capacity_tokens=self.cfg.capacity_tokens,
            samples=self.samples,
        )

    def report_device(self) -> MetricsReport:
        """compute_metrics (engine.py:132-211) evaluated on the device
        (co_metrics): per-request aggregation, exact integer
        sums, numpy-pairwise normalized-latency sum and radix-selected order
        statistics; only the interpolation below and the per-iteration
        utilization samples (already streamed to the host) are host work.
        Equal to ``run()``'s report field for field."""
        s = self._scalars()
        raw = N.CoMetricsRaw()
        N.check(self._lib.co_metrics(self._h, C.byref(raw)), "co_metrics")
        n = self._n
        makespan = max(0, int(s.now_us) - int(s.first_arrival_us))
        span_s = makespan / US_PER_S if makespan > 0 else 0.0

        def pct(lst: int, total) -> Dict[str, float]:
            return pct_from_order_stats(int(raw.count[lst]), [float(v) for v in raw.order_stat[lst]], total)

        samples = self.samples
        cap = self.cfg.capacity_tokens
        if len(samples):
            util = float(np.mean([fp / cap for fp, _ in samples]))
            frag = float(np.mean([(fp - u) / cap for fp, u in samples]))
        else:
            util = frag = 0.0
        done = int(raw.completed)

        def mean(total, cnt):
            return float(total) / cnt if cnt else 0.0

        return MetricsReport(
            policy=self.cfg.sched.policy, seed=self.cfg.seed, num_requests=n, completed=done,
            makespan_us=makespan, ttft_us=pct(0, raw.sum_ttft), tbt_us=pct(1, raw.sum_gap),
            ttft_attainment=raw.ok_ttft / n if n else 0.0, tbt_attainment=raw.ok_tbt / n if n else 0.0,
            normalized_us_per_token=pct(2, raw.norm_sum),
            preemption_total=int(raw.preemption_total), preempted_requests=int(raw.preempted),
            preemption_time_us=pct(3, raw.sum_ptime),
            throughput_rps=done / span_s if span_s else 0.0,
            throughput_tps=int(raw.generated) / span_s if span_s else 0.0,
            kvc_utilization_mean=util, kvc_fragmentation_mean=frag,
            waiting_us_mean=mean(raw.sum_wait, done), execution_us_mean=mean(raw.sum_exec, done),
            preemption_us_mean=mean(raw.sum_pdec, done),
        )

    def last_device_ms(self) -> float:
        ms = C.c_double()
        N.check(self._lib.co_last_device_ms(self._h, C.byref(ms)), "co_last_device_ms")
        return float(ms.value)

    def _preempt(self, rid: int, strategy: Strategy, now_us: int, cause: str = "plan") -> None:
        """White-box hook matching engine.py:360-384."""
        self._dirty()
        N.check(self._lib.co_preempt(self._h, self._idx_of[rid], STRATEGY_CODE[strategy], now_us,
                                     CAUSE_CODE[cause]), "co_preempt")

    def block_tables(self):
        """N1 readback: ({req_id: [page ids]}, free stack bottom..top)."""
        lens = np.empty(max(self._n, 1), dtype=np.int32)
        npg = self.cfg.capacity_tokens // self.cfg.sched.small_block_b
        pages = np.empty(max(npg, 1), dtype=np.int32)
        free = np.empty(max(npg, 1), dtype=np.int32)
        nf = C.c_int32()
        N.check(self._lib.co_read_block_tables(self._h, _ptr(lens, C.c_int32), _ptr(pages, C.c_int32), npg,
                                               _ptr(free, C.c_int32), C.byref(nf)), "co_read_block_tables")
        out, w = {}, 0
        for k in range(self._n):
            if lens[k]:
                out[self._rid[k]] = pages[w:w + lens[k]].tolist()
                w += int(lens[k])
        return out, free[:nf.value].tolist()

    # -- N2/N3 data plane --------------------------------------------------------

    def data_stats(self) -> Dict[str, int]:
        st = np.zeros(8, dtype=np.int64)
        N.check(self._lib.co_data_stats(self._h, _ptr(st, C.c_int64)), "co_data_stats")
        keys = ("swap_out_bytes", "swap_in_bytes", "fill_bytes", "move_bytes", "decode_steps",
                "decode_member_steps", "decode_ctx_tokens")
        return dict(zip(keys, (int(v) for v in st)))

    def swap_io_stats(self) -> Dict[str, float]:
        """The split swap I/O's device-timed totals (k_swapio beside the decode):
        bytes each way over the host link, device seconds, launches."""
        st = np.zeros(6, dtype=np.int64)
        N.check(self._lib.co_swap_io_stats(self._h, _ptr(st, C.c_int64)), "co_swap_io_stats")
        out, inn, ns, launches, split, ctas = (int(v) for v in st)
        return {"bytes_out": out, "bytes_in": inn, "device_s": ns * 1e-9, "launches": launches,
                "gbs": (out + inn) / (ns * 1e-9) / 1e9 if ns else 0.0, "split": bool(split), "ctas": ctas}

    # -- N4 global reserve telemetry ---------------------------------------------

    def attach_nccl(self, uid: bytes, nranks: int, rank: int) -> None:
        buf = (C.c_uint8 * len(uid)).from_buffer_copy(uid)
        N.check(self._lib.co_attach_nccl(self._h, buf, nranks, rank), "co_attach_nccl")

    def global_reserve(self) -> Tuple[int, int, int]:
        """(sum of free_tokens, sum of reserved_blocks_current, all-reduce calls)."""
        out = np.zeros(2, dtype=np.int64)
        calls = C.c_int64()
        N.check(self._lib.co_global_reserve(self._h, _ptr(out, C.c_int64), C.byref(calls)), "co_global_reserve")
        return int(out[0]), int(out[1]), int(calls.value)

    def set_decode(self, on: bool) -> None:
        N.check(self._lib.co_set_decode(self._h, int(on)), "co_set_decode")

    def swap_bench(self, ntok: int, iters: int = 5) -> Tuple[float, float]:
        """(gather ms, scatter ms) of ntok tokens through the engine's data kernel."""
        a, b = C.c_double(), C.c_double()
        N.check(self._lib.co_swap_bench(self._h, ntok, iters, C.byref(a), C.byref(b)), "co_swap_bench")
        return float(a.value), float(b.value)

    def kv_verify(self) -> Tuple[int, int]:
        bad, chk = C.c_int64(), C.c_int64()
        N.check(self._lib.co_kv_verify(self._h, C.byref(bad), C.byref(chk)), "co_kv_verify")
        return int(bad.value), int(chk.value)

    def last_decode(self):
        """(member req_ids, ctx lengths, out[m][layer][q_head][128] fp32, step id)."""
        kv = self.kv
        cap = min(self._n, 4096)
        mem = np.empty(max(cap, 1), dtype=np.int32)
        ctx = np.empty(max(cap, 1), dtype=np.int32)
        out = np.empty((max(cap, 1), kv.layers, kv.q_heads, kv.head_dim), dtype=np.float32)
        n, sid = C.c_int64(), C.c_int64()
        N.check(self._lib.co_read_decode(self._h, _ptr(mem, C.c_int32), _ptr(ctx, C.c_int32),
                                         out.ctypes.data_as(C.POINTER(C.c_float)), cap, C.byref(n), C.byref(sid)),
                "co_read_decode")
        k = int(n.value)
        return [self._rid[i] for i in mem[:k]], ctx[:k].copy(), out[:k].copy(), int(sid.value)

    def check_invariants(self) -> None:
        N.check(self._lib.co_check_invariants(self._h), "check_invariants")

    # -- host views ------------------------------------------------------------

    def _drain(self) -> None:
        """Move the device append log (events, iteration members, utilization
        samples) into the host lists in one library call.  After a step() the
        library serves it from the step graph's pinned mirror, so this is
        host-only work (ctypes buffers: no numpy per call)."""
        cnt = self._cnt
        while True:
            if self._evbuf is None:
                ne, nm, ns = (max(1024, int(x)) for x in cnt)
                nm = max(nm, 16384)
                self._evbuf = (N.CoEvent * ne)()
                self._membuf = (C.c_int32 * (2 * nm))()
                self._sbuf = (C.c_int64 * (2 * ns))()
                self._drain_args = (self._h, self._evbuf, ne, self._membuf, nm, self._sbuf, ns, self._cnt)
                self._step_args = {}  # (they point at these buffers)
                self._mem_addr = C.addressof(self._membuf)
                self._ev_addr = C.addressof(self._evbuf)
            rc = self._lib.co_drain_log(*self._drain_args)
            if rc != N.CO_EAGAIN:
                break
            self._evbuf = None  # grow to the sizes returned in cnt and retry
        N.check(rc, "co_drain_log")
        self._take_log()

    def _take_log(self) -> None:
        cnt = self._cnt
        ne, ns = cnt[0], cnt[2]
        if ne:
            self._events.extend(self._convert(ne, None))
        if ns:
            it = iter(self._sbuf[:2 * ns])
            self._samples.extend(zip(it, it))
        self._sc = None

    def _convert(self, n: int, mem: np.ndarray) -> List[dict]:
        """Device event records -> the reference's event dicts (engine.py:
        353, 376-383, 407, 512-518, 533), built by the _hostlog extension."""
        return (_hostlog or _load_hostlog()).convert(self._ev_addr, n, self._mem_addr, self._rid, _STRATEGY_NAMES,
                                                     _CAUSE_NAMES)

    @property
    def events(self) -> List[dict]:
        if not self._log_clean:
            self._drain()
        return self._events

    @property
    def samples(self) -> List[Tuple[int, int]]:
        self._drain()
        return self._samples

    @property
    def requests(self) -> Dict[int, Request]:
        """The caller's Request objects (engine.py:239), their ``state`` current
        as of the last step (the reference transitions them in-step,
        core.py:113-130; here one STATE readback after a step, on access)."""
        if self._req_stale:
            self.requests_view()
        return self._requests

    def requests_view(self) -> Dict[int, Request]:
        st = self._field("STATE")
        reqs = self._requests
        for k, r in enumerate(self._rid):
            reqs[r].state = STATE_FROM_CODE[int(st[k])]
        self._req_stale = False
        return reqs

    @property
    def runtimes(self) -> Dict[int, RequestRuntime]:
        self.requests_view()
        f = self._field
        cols = {name: f(name).tolist() for name in (
            "GENERATED", "ALLOCATED_KVC", "USED", "FIRST_TOKEN", "LAST_TOKEN", "MAX_TBT",
            "PREEMPTION_COUNT", "PREEMPTION_TIME", "KV_NEED", "PREFILL_DONE", "READY_AT",
            "PREEMPT_STARTED", "SWAP_OUT_DONE", "LAST_STRATEGY", "FIRST_START", "COMPLETION",
            "PREDICTED", "ESTIMATED", "STATE")}
        offs = np.empty(self._n + 1, dtype=np.int64)
        times = np.empty(max(1, int(self._tok_total())), dtype=np.int64)
        N.check(self._lib.co_read_token_times(self._h, _ptr(offs, C.c_int64), _ptr(times, C.c_int64)),
                "co_read_token_times")
        w = self.cfg.predictor.bin_width
        out = _Runtimes()
        none = lambda v: None if v < 0 else v  # noqa: E731
        for k, r in enumerate(self._rid):
            g = cols["GENERATED"][k]
            est = None
            if cols["STATE"][k] != 0:
                p, e = cols["PREDICTED"][k], cols["ESTIMATED"][k]
                lo, hi = bin_of(p, w)
                est = LengthEstimate(predicted_len=p, range_lo=lo, range_hi=hi,
                                     direction=Direction.UNDER if self._under[k] else Direction.OVER,
                                     confidence=self.confidence, padding=self.padding, estimated_len=e)
            ls = cols["LAST_STRATEGY"][k]
            out[r] = RequestRuntime(
                generated=g, allocated_kvc=cols["ALLOCATED_KVC"][k], used_kvc=cols["USED"][k],
                first_token_at_us=none(cols["FIRST_TOKEN"][k]), last_token_at_us=none(cols["LAST_TOKEN"][k]),
                max_tbt_us=cols["MAX_TBT"][k], preemption_count=cols["PREEMPTION_COUNT"][k],
                preemption_time_us=cols["PREEMPTION_TIME"][k], estimate=est, kv_need=cols["KV_NEED"][k],
                prefill_done=cols["PREFILL_DONE"][k], ready_at_us=cols["READY_AT"][k],
                preempt_started_us=cols["PREEMPT_STARTED"][k], swap_out_done_us=cols["SWAP_OUT_DONE"][k],
                last_strategy=STRATEGY_FROM_CODE.get(ls), first_start_us=none(cols["FIRST_START"][k]),
                completion_us=none(cols["COMPLETION"][k]),
                token_times_us=times[offs[k]:offs[k] + g].tolist(),
            )
        # present in the caller's input order like the reference dicts
        return {r: out[r] for r in self._input_order}

    def _tok_total(self) -> int:
        return int(sum(r.true_output_len for r in self._requests.values()))
