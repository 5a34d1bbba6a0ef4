"""CPU oracle for the CacheOPT per-iteration hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2503_13773_b200`` imports or
calls this module; only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may use it, and
only as the checker or the timed CPU baseline.

What it is: an independent restatement of the reference simulator's engine
loop for the ``cacheopt`` policy (``/root/reference/pkg/src/kvcsim``), written
over a structure-of-arrays request table instead of per-request objects.
Every function cites the reference ``file:line`` it restates.  The restatement
is pinned against the reference itself: ``tests/golden/`` holds event logs and
final states produced by running the unmodified reference on seeded traces
(``oracle/make_golden.py``), and ``tests/test_oracle_golden.py`` replays them.

Inputs are duck-typed: ``requests`` are objects with ``id, arrival_us,
prompt_len, true_output_len, slo_ttft_us, slo_tbt_us``; ``cfg`` is any object
shaped like the reference ``EngineConfig`` (``engine.py:66-89``), so the same
oracle runs with the reference's dataclasses here and with the product's
mirror dataclasses on the GPU box.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional, Tuple

import numpy as np

# lifecycle codes (core.py:26-30); PENDING = not yet arrived
PENDING, WAITING, RUNNING, PREEMPTED, COMPLETED = 0, 1, 2, 3, 4
SWAP, RECOMPUTE = 0, 1
STRATEGY_NAME = {SWAP: "swap", RECOMPUTE: "recompute"}
NO_PROGRESS_LIMIT = 1_000_000  # engine.py:62


# ---------------------------------------------------------------------------
# scalar arithmetic restated from the reference (float paths kept in IEEE
# double exactly as Python evaluates them)


def to_us(ms: float) -> int:
    """core.py:21-23 -- ms to integer us, half up."""
    return math.floor(ms * 1000 + 0.5)


def iter_ms(cfg, batch_tokens: int) -> float:
    """costmodel.py:51-55."""
    c = cfg.iter_cost
    return c.base_ms + c.per_token_ms * batch_tokens


def swap_ms(model, s) -> float:
    """preemption.py:94-95 (SwapModel.predict)."""
    return model.gamma_s * s + model.delta_s


def recompute_ms(model, s) -> float:
    """preemption.py:115-116 (RecomputeModel.predict)."""
    return model.alpha_r * s ** model.beta_r + model.kappa_r * s + model.eps_r


def sweet_spot_s_star(swp, rec, s_max: int = 1_000_000) -> int:
    """preemption.py:176-195 bisection, plus the dominance fallback of
    scheduler.py:381-393."""
    def diff(s):
        return recompute_ms(rec, s) - swap_ms(swp, s)
    lo, hi = 1, s_max
    if diff(lo) > 0 or diff(hi) <= 0:
        return 0 if recompute_ms(rec, 1) > swap_ms(swp, 1) else (1 << 62)
    while hi - lo > 1:
        mid = (lo + hi) // 2
        if diff(mid) <= 0:
            lo = mid
        else:
            hi = mid
    return lo


def confidence_for(cfg, requests_sorted) -> float:
    """engine.py:251-266 and estimation.py:102-107."""
    if cfg.fixed_confidence is not None:
        return cfg.fixed_confidence
    if requests_sorted:
        first = requests_sorted[0].arrival_us
        span = requests_sorted[-1].arrival_us - first
        rate = (len(requests_sorted) - 1) / (span / 1_000_000) if span > 0 else 0.0
    else:
        rate = 0.0
    pol = cfg.confidence
    raw = pol.alpha / (1.0 + pol.beta * rate)
    return min(pol.clamp_hi, max(pol.clamp_lo, raw))


def padding_tokens(pred_cfg, confidence: float) -> int:
    """estimation.py:110-119 with range hi-lo = bin_width-1 (:94-95, :142)."""
    if pred_cfg.fixed_padding is not None:
        return pred_cfg.fixed_padding
    width = pred_cfg.bin_width - 1
    raw = width * math.sqrt(-math.log(1.0 - confidence) / 2.0)
    return min(width, math.floor(raw + 0.5))


def draw_estimate_noise(pred_cfg, rng) -> Tuple[int, bool]:
    """The RNG consumption of one ``predict`` call (estimation.py:76-99):
    the error draw, then a flip draw only when direction accuracy < 1."""
    if pred_cfg.error_dist == "zero":
        err = 0
    elif pred_cfg.error_dist == "uniform":
        s = int(pred_cfg.error_scale)
        err = int(rng.integers(-s, s + 1)) if s > 0 else 0
    else:
        err = math.floor(float(rng.normal(0.0, pred_cfg.error_scale)) + 0.5)
    flip = False
    if pred_cfg.direction_accuracy < 1.0:
        flip = bool(rng.random() < 1.0 - pred_cfg.direction_accuracy)
    return err, flip


def estimate_from_noise(true_len: int, err: int, flip: bool, pad: int) -> Tuple[int, int]:
    """estimation.py:85-99, 122-128: (predicted, estimated)."""
    pred = max(1, true_len - err)
    under = true_len >= pred
    if flip:
        under = not under
    est = pred + pad if under else max(1, pred - pad)
    return pred, est


def split_largest_remainder_inverted(demands: List[Tuple[int, int, int, int]], supply: int) -> Dict[int, int]:
    """scheduler.py:211-243 with ``invert=True`` (weights 1/(rt*p), :233),
    restated with ``Fraction`` exactly as the reference computes it (the
    shares have no small common denominator)."""
    from fractions import Fraction
    if supply < 0:
        raise ValueError("a_prime must be >= 0")
    live = [d for d in demands if d[1] > 0]
    if not live:
        return {}
    if sum(d[1] for d in live) <= supply:
        return {d[0]: d[1] for d in live}
    w = {d[0]: 1 / Fraction(max(1, d[2]) * max(1, d[3])) for d in live}
    W = sum(w.values())
    share = {r: Fraction(supply) * x / W for r, x in w.items()}
    q = {r: int(x) for r, x in share.items()}
    left = supply - sum(q.values())
    for rid in sorted(share, key=lambda r: (-(share[r] - q[r]), r))[:left]:
        q[rid] += 1
    return q


def split_largest_remainder(demands: List[Tuple[int, int, int, int]], supply: int) -> Dict[int, int]:
    """scheduler.py:211-243 without ``Fraction``: every share has the common
    denominator W = sum(w), so floor(a*w_i/W) and the remainder a*w_i mod W
    reproduce the rational floors and the largest-remainder order exactly.

    demands: (req_id, m_tokens, rt_us, prompt_len)."""
    if supply < 0:
        raise ValueError("a_prime must be >= 0")
    live = [d for d in demands if d[1] > 0]
    if not live:
        return {}
    if sum(d[1] for d in live) <= supply:
        return {d[0]: d[1] for d in live}
    w = [max(1, d[2]) * max(1, d[3]) for d in live]
    W = sum(w)
    q = {}
    r = {}
    for d, wi in zip(live, w):
        q[d[0]], r[d[0]] = divmod(supply * wi, W)
    left = supply - sum(q.values())
    for rid in sorted(q, key=lambda k: (-r[k], k))[:left]:
        q[rid] += 1
    return q


# ---------------------------------------------------------------------------
# the engine


class CacheOptOracle:
    """engine.py:222-672 for policy ``cacheopt`` (scheduler.py:408-753),
    over a structure-of-arrays request table indexed by arrival rank."""

    def __init__(self, requests, cfg):
        ids = [r.id for r in requests]
        if len(set(ids)) != len(ids):
            raise ValueError("request ids must be unique")
        if cfg.sched.policy not in ("cacheopt", "vllm_block", "sarathi_chunked", "rlp", "s3"):
            raise ValueError(f"unknown policy {cfg.sched.policy!r}")
        self.cfg = cfg
        reqs = sorted(requests, key=lambda r: (r.arrival_us, r.id))  # engine.py:241
        n = self.n = len(reqs)
        self.rid = [int(r.id) for r in reqs]
        self.idx_of = {r: i for i, r in enumerate(self.rid)}
        self.input_order = [self.idx_of[int(r.id)] for r in requests]  # engine.py:239 dict order
        I64 = np.int64
        self.arr = np.array([r.arrival_us for r in reqs], dtype=I64)
        self.prompt = np.array([r.prompt_len for r in reqs], dtype=I64)
        self.tout = np.array([r.true_output_len for r in reqs], dtype=I64)
        self.slo_ttft = np.array([r.slo_ttft_us for r in reqs], dtype=I64)
        self.slo_tbt = np.array([r.slo_tbt_us for r in reqs], dtype=I64)
        # runtime (core.py:72-94)
        self.state = np.zeros(n, dtype=np.int8)
        self.gen = np.zeros(n, dtype=I64)
        self.used = np.zeros(n, dtype=I64)
        self.kv_need = self.prompt.copy()
        self.prefill = np.zeros(n, dtype=I64)
        self.pcount = np.zeros(n, dtype=I64)
        self.ptime = np.zeros(n, dtype=I64)
        self.first_tok = np.full(n, -1, dtype=I64)
        self.last_tok = np.full(n, -1, dtype=I64)
        self.max_tbt = np.zeros(n, dtype=I64)
        self.ready_at = np.zeros(n, dtype=I64)
        self.pstart = np.zeros(n, dtype=I64)
        self.swap_done = np.zeros(n, dtype=I64)
        self.last_strat = np.full(n, -1, dtype=I64)
        self.first_start = np.full(n, -1, dtype=I64)
        self.completion = np.full(n, -1, dtype=I64)
        self.alloc_kvc = np.zeros(n, dtype=I64)
        self.pred = np.zeros(n, dtype=I64)
        self.est = np.zeros(n, dtype=I64)
        self.token_times: List[List[int]] = [[] for _ in range(n)]
        # pool records (kvc.py:44-52, 55-84)
        sc = cfg.sched
        self.bs = sc.small_block_b                       # engine.py:236
        self.capacity = cfg.capacity_tokens
        self.buffer_b = sc.buffer_b
        self.stacking = cfg.allow_stacking
        if cfg.reserved_blocks * self.bs > self.capacity:
            raise ValueError("reserve exceeds capacity")
        self.rsv_target = cfg.reserved_blocks
        self.rsv_cur = cfg.reserved_blocks
        self.holds = np.zeros(n, dtype=bool)
        self.granted = np.zeros(n, dtype=I64)
        self.host = np.full(n, -1, dtype=I64)
        self.off = np.zeros(n, dtype=I64)
        self.rsv = np.zeros(n, dtype=I64)
        self.rec_seq = np.zeros(n, dtype=I64)
        self.guests: Dict[int, List[int]] = {}
        # N1 block tables (defined by this framework):
        # LIFO free stack of page ids, popped 0, 1, 2, ... initially
        self.n_pages = self.capacity // self.bs
        self.free_pages: List[int] = list(range(self.n_pages - 1, -1, -1))
        self.tables: Dict[int, List[int]] = {}
        self.seq = 0
        self.fp_sum = 0
        self.granted_sum = 0
        self.used_sum = 0
        # engine scalars
        self.claims: Dict[int, int] = {}  # provider idx -> waiter idx
        self.events: List[dict] = []
        self.samples: List[Tuple[int, int]] = []
        self.iters = 0
        self.gen_total = 0
        self.next_pending = 0
        self.n_live = 0
        self.stalled = False
        if n:
            self.first_arrival = int(self.arr[0])
            last = int(self.arr[-1])
            span = last - self.first_arrival
            self.horizon = last + cfg.horizon_factor * max(span, 1_000_000)
        else:
            self.first_arrival = 0
            self.horizon = 0
        self.now = self.first_arrival
        self.confidence = confidence_for(cfg, reqs)
        self.pad = padding_tokens(cfg.predictor, self.confidence)
        self.rng = np.random.default_rng([cfg.seed, 3])            # engine.py:267
        self.t_i = to_us(iter_ms(cfg, sc.token_budget))            # engine.py:268-270
        tr = cfg.truth
        self.s_star = sweet_spot_s_star(tr.swap_true, tr.recompute_true)
        self.record_events = cfg.record_events
        self._ids_np = np.array(self.rid, dtype=np.int64)

    # -- pool (kvc.py) ------------------------------------------------------

    def _fp(self, t):
        bs = self.bs
        return ((t + bs - 1) // bs) * bs

    def free_tokens(self):
        """kvc.py:92-98."""
        return self.capacity - self.rsv_cur * self.bs - self.fp_sum

    def _pop_pages(self, i, k):
        tab = self.tables.setdefault(i, [])
        for _ in range(k):
            tab.append(self.free_pages.pop())

    def _push_pages(self, i):
        for pg in reversed(self.tables.pop(i, [])):
            self.free_pages.append(pg)

    def _new_record(self, i, granted, host=-1, off=0):
        self.holds[i] = True
        self.granted[i] = granted
        self.host[i] = host
        self.off[i] = off
        self.rsv[i] = 0
        self.seq += 1
        self.rec_seq[i] = self.seq  # dict insertion order of kvc.py:82

    def _drop_record(self, i):
        self.holds[i] = False
        self.used_sum -= int(self.used[i])
        self.guests.pop(i, None)

    def eff_alloc(self, i):
        """engine.py:275-282."""
        if not self.holds[i]:
            return 0
        g = int(self.granted[i])
        gl = self.guests.get(i)
        if gl:
            return min(g, min(int(self.off[x]) for x in gl))
        return g

    def release_gain(self, i):
        """kvc.py:142-152."""
        if self.host[i] >= 0:
            return 0
        freed = self._fp(int(self.granted[i]))
        for gid in self.guests.get(i, ()):
            freed -= self._fp(int(self.granted[gid]))
        refill = min(int(self.rsv[i]), self.rsv_target - self.rsv_cur)
        return freed - refill * self.bs

    def pool_allocate(self, i, n):
        """kvc.py:156-167; False on Shortfall or contract violation."""
        if n < 1 or self.holds[i]:
            return False
        fp = self._fp(n)
        if fp > self.free_tokens():
            return False
        self._new_record(i, n)
        self.fp_sum += fp
        self.granted_sum += n
        self._pop_pages(i, fp // self.bs)
        return True

    def find_host(self, triples, prompt, out):
        """kvc.py:169-200 -> (host, start_offset) or None."""
        b = self.buffer_b
        need = prompt + out
        best = None
        for h, a_j, u_j in triples:
            if not self.holds[h] or self.host[h] >= 0:
                continue
            gl = self.guests.get(h)
            if gl and not self.stacking:
                continue
            end = min(int(self.off[g]) for g in gl) if gl else a_j
            slack = end - (u_j + out) - need
            if slack < b:
                continue
            key = (a_j - u_j, self.rid[h])
            if best is None or key < best[0]:
                best = (key, h, end - need)
        return None if best is None else (best[1], best[2])

    def pool_embed(self, i, n, host, start):
        """kvc.py:202-227."""
        if n < 1 or self.holds[i] or not self.holds[host]:
            return False
        if self.host[host] >= 0 or i == host:
            return False
        gl = self.guests.get(host, [])
        if gl and not self.stacking:
            return False
        if start < 0 or start + n > self.granted[host]:
            return False
        for g in gl:
            if not (start + n <= self.off[g] or self.off[g] + self.granted[g] <= start):
                return False
        self._new_record(i, n, host=host, off=start)
        self.guests.setdefault(host, []).append(i)
        self.granted_sum += n
        return True

    def pool_draw_reserved(self, i, nb):
        """kvc.py:229-249."""
        if nb < 1 or nb > self.rsv_cur:
            return False
        if not self.holds[i]:
            self._new_record(i, 0)
        if self.host[i] >= 0:
            return False
        tokens = nb * self.bs
        self.rsv_cur -= nb
        self.rsv[i] += nb
        g = int(self.granted[i])
        old = self._fp(g) if g else 0
        self.granted[i] = g + tokens
        dfp = self._fp(g + tokens) - old
        self.fp_sum += dfp
        self.granted_sum += tokens
        self._pop_pages(i, dfp // self.bs)
        return True

    def pool_grow(self, i, n):
        """kvc.py:251-281."""
        if n < 1 or not self.holds[i]:
            return False
        g = int(self.granted[i])
        h = int(self.host[i])
        if h < 0:
            delta = self._fp(g + n) - self._fp(g)
            if delta > self.free_tokens():
                return False
            self.granted[i] = g + n
            self.fp_sum += delta
            self.granted_sum += n
            self._pop_pages(i, delta // self.bs)
            return True
        floor = int(self.used[h]) + self.buffer_b
        for gid in self.guests.get(h, ()):
            if gid != i and self.off[gid] < self.off[i]:
                floor = max(floor, int(self.off[gid] + self.granted[gid]))
        if n > int(self.off[i]) - floor:
            return False
        self.off[i] -= n
        self.granted[i] = g + n
        self.granted_sum += n
        return True

    def pool_promote(self, i):
        """kvc.py:283-297."""
        fp = self._fp(int(self.granted[i]))
        if fp > self.free_tokens():
            return False
        h = int(self.host[i])
        self.guests[h].remove(i)
        if not self.guests[h]:
            del self.guests[h]
        self.host[i] = -1
        self.off[i] = 0
        self.fp_sum += fp
        self._pop_pages(i, fp // self.bs)
        return True

    def pool_release(self, i):
        """kvc.py:299-324."""
        h = int(self.host[i])
        if h >= 0:
            gl = self.guests.get(h)
            if gl is not None:
                gl.remove(i)
                if not gl:
                    del self.guests[h]
            self.granted_sum -= int(self.granted[i])
            self.host[i] = -1
            self._drop_record(i)
            return
        self._push_pages(i)
        if len(self.guests.get(i, ())) > 1:
            self.multi_rehomes = getattr(self, "multi_rehomes", 0) + 1  # stacked guests re-homed at once
        for gid in self.guests.get(i, ()):
            self.host[gid] = -1
            self.off[gid] = 0
            gfp = self._fp(int(self.granted[gid]))
            self.fp_sum += gfp
            self._pop_pages(gid, gfp // self.bs)
        self.fp_sum -= self._fp(int(self.granted[i]))
        self.granted_sum -= int(self.granted[i])
        refill = min(int(self.rsv[i]), self.rsv_target - self.rsv_cur)
        self.rsv_cur += refill
        self._drop_record(i)

    def set_used(self, i, u):
        """kvc.py:326-332."""
        if u < 0 or u > self.granted[i]:
            raise ValueError(f"request {self.rid[i]}: used {u} outside [0, {self.granted[i]}]")
        self.used_sum += u - int(self.used[i])
        self.used[i] = u

    def block_tables(self):
        """N1 state: ({req_id: pages}, free stack bottom..top)."""
        return ({self.rid[i]: list(t) for i, t in sorted(self.tables.items()) if t}, list(self.free_pages))

    def check_invariants(self):
        """kvc.py:336-375."""
        owners = np.nonzero(self.holds)[0]
        fp = sum(self._fp(int(self.granted[i])) for i in owners if self.host[i] < 0)
        if fp != self.fp_sum:
            raise ValueError("footprint drift")
        if self.free_tokens() < 0:
            raise ValueError("free tokens negative")
        if not 0 <= self.rsv_cur <= self.rsv_target:
            raise ValueError("reserve out of range")
        # N1: standalone records own exactly fp(granted)/bs distinct pages
        seen = set(self.free_pages)
        if len(seen) != len(self.free_pages):
            raise ValueError("duplicate free page")
        for i, t in self.tables.items():
            want = self._fp(int(self.granted[i])) // self.bs if (self.holds[i] and self.host[i] < 0) else 0
            if len(t) != want:
                raise ValueError(f"table of {self.rid[i]} has {len(t)} pages, footprint needs {want}")
            for pg in t:
                if pg in seen:
                    raise ValueError("page owned twice")
                seen.add(pg)
        if len(seen) != self.n_pages or self.fp_sum // self.bs != self.n_pages - len(self.free_pages):
            raise ValueError("page conservation")
        for i in owners:
            if self.used[i] > self.granted[i]:
                raise ValueError("used exceeds granted")
            h = self.host[i]
            if h >= 0:
                if not self.holds[h] or i not in self.guests.get(int(h), []):
                    raise ValueError("guest detached")
                if self.off[i] < 0 or self.off[i] + self.granted[i] > self.granted[h]:
                    raise ValueError("guest exceeds host region")
            gl = self.guests.get(int(i))
            if gl:
                prev = int(self.used[i])
                for s, e in sorted((int(self.off[g]), int(self.off[g] + self.granted[g])) for g in gl):
                    if s < prev:
                        raise ValueError("guest overlap")
                    prev = e

    # -- events -------------------------------------------------------------

    def _ev(self, **kw):
        if self.record_events:
            self.events.append(kw)

    # -- lifecycle (engine.py:344-433) ----------------------------------------

    def _admit_arrivals(self):
        """engine.py:344-353: arrivals in (arrival, id) order draw their
        estimate noise from the shared stream in that order."""
        pc = self.cfg.predictor
        while self.next_pending < self.n and self.arr[self.next_pending] <= self.now:
            i = self.next_pending
            self.next_pending += 1
            err, flip = draw_estimate_noise(pc, self.rng)
            self.pred[i], self.est[i] = estimate_from_noise(int(self.tout[i]), err, flip, self.pad)
            self.state[i] = WAITING
            self.n_live += 1
            self._ev(ev="arrive", t=int(self.arr[i]), req=self.rid[i])

    def _strategy(self, i):
        """engine.py:355-358 / scheduler.py:357-359 / preemption.py:198-200."""
        return SWAP if max(1, int(self.used[i])) > self.s_star else RECOMPUTE

    def _preempt(self, i, strat, now, cause="plan"):
        """engine.py:360-384."""
        if self.state[i] != RUNNING:
            return
        self.state[i] = PREEMPTED
        self.pcount[i] += 1
        self.last_strat[i] = strat
        u = int(self.used[i])
        restored = max(1, u)
        self.pstart[i] = now
        self.prefill[i] = u
        self.kv_need[i] = max(int(self.kv_need[i]), u)
        if strat == SWAP:
            self.swap_done[i] = now + to_us(swap_ms(self.cfg.truth.swap_true, restored) / 2.0)
        else:
            self.swap_done[i] = 0
        if self.holds[i]:
            self.pool_release(i)
        self.used[i] = 0
        self.alloc_kvc[i] = 0
        self.claims.pop(i, None)
        for p in [p for p, w in self.claims.items() if w == i]:
            del self.claims[p]
        self._ev(ev="preempt", t=now, req=self.rid[i], strategy=STRATEGY_NAME[strat],
                 kv=restored, cause=cause)

    def _readmit(self, i):
        """engine.py:386-402."""
        self.state[i] = RUNNING
        restored = max(1, int(self.prefill[i]))
        tr = self.cfg.truth
        if self.last_strat[i] == SWAP:
            half = to_us(swap_ms(tr.swap_true, restored) / 2.0)
            self.ready_at[i] = max(self.now, int(self.swap_done[i])) + half
        else:
            self.ready_at[i] = self.now + to_us(recompute_ms(tr.recompute_true, restored))
        self.ptime[i] += self.ready_at[i] - self.pstart[i]
        u = min(int(self.prefill[i]), int(self.granted[i]))
        self.set_used(i, u)
        self._ev(ev="readmit", t=self.now, req=self.rid[i], ready_at=int(self.ready_at[i]))

    def _complete(self, i, now):
        """engine.py:404-417."""
        self.state[i] = COMPLETED
        self.completion[i] = now
        if self.holds[i]:
            self.pool_release(i)
        self.n_live -= 1
        self._ev(ev="complete", t=now, req=self.rid[i])
        for p in [p for p, w in self.claims.items() if w == i]:
            del self.claims[p]
        w = self.claims.pop(i, None)
        if w is not None and self.state[w] in (WAITING, RUNNING, PREEMPTED):
            self._fulfill_claim(w)

    def _fulfill_claim(self, w):
        """engine.py:419-433."""
        if self.state[w] != RUNNING or not self.holds[w]:
            return
        target = max(int(self.used[w]), int(self.kv_need[w])) + max(0, int(self.est[w] - self.gen[w]))
        residual = target - int(self.granted[w])
        if residual > 0 and self.pool_grow(w, residual):
            self.alloc_kvc[w] = self.granted[w]

    # -- the planner (scheduler.py:408-753) ---------------------------------

    def _rt(self, i):
        """scheduler.py:108-113 over engine.py:288-295 slacks."""
        if self.first_tok[i] < 0:
            return int(self.slo_ttft[i]) - (self.now - int(self.arr[i]))
        return int(self.slo_tbt[i]) - (self.now - int(self.last_tok[i]))

    # -- baseline planners (scheduler.py:760-936) ---------------------------

    def _baseline_views(self):
        live = np.nonzero((self.state >= WAITING) & (self.state <= PREEMPTED))[0]
        running = [int(i) for i in live if self.state[i] == RUNNING]
        waiting = [int(i) for i in live if self.state[i] != RUNNING]  # _live order (engine.py:321-324)
        eff = {i: self.eff_alloc(i) for i in running + waiting}
        ready = {i: self.state[i] != RUNNING or self.now >= self.ready_at[i] for i in running + waiting}
        return running, waiting, eff, ready

    def _cost(self, i, grant):
        """_FreeTracker.alloc_cost (scheduler.py:350-354)."""
        if self.holds[i] and self.host[i] >= 0:
            return 0
        h = int(self.granted[i]) if self.holds[i] else 0
        return self._fp(h + grant) - self._fp(h)

    def _fcfs(self, waiting):
        """scheduler.py:760-766: preempted first, FCFS (index = (arrival, id)) within each."""
        return [i for i in waiting if self.state[i] == PREEMPTED] + [i for i in waiting if self.state[i] != PREEMPTED]

    def _plan_dict(self, members, preempt, actions):
        bt = sum(t for _, t in members)
        return dict(members=members, preempt=preempt, actions=actions, claims=[], deferred=[],
                    overflow=bt > self.cfg.sched.token_budget, batch_tokens=bt)

    def plan_vllm_block(self, chunked=False):
        """scheduler.py:769-838 (chunked: sarathi_chunked)."""
        sc = self.cfg.sched
        running, waiting, eff, ready = self._baseline_views()
        running = [i for i in running if ready[i]]
        free = self.free_tokens()
        step = sc.vllm_block_tokens
        budget = sc.token_budget
        members, preempt, actions = [], [], []
        removed = set()
        returned = {i: eff[i] < int(self.used[i]) + 1 for i in running}  # every view here is RUNNING
        for i in running:  # sorted by (arrival, id) = index order
            if not returned[i] or i in removed:
                continue
            while True:
                cost = self._cost(i, step)
                if cost <= free:
                    actions.append(("grow", i, step, 0, -1, 0))
                    free -= cost
                    break
                cands = [x for x in running if x not in removed and self.holds[x]]
                if not cands:
                    break
                victim = cands[-1]  # max (arrival, id)
                preempt.append((victim, RECOMPUTE))
                removed.add(victim)
                free += self.release_gain(victim)
                if victim == i:
                    break
        grown = {a[1] for a in actions}
        for i in running:
            if i in removed or self.state[i] != RUNNING:
                continue
            if self.prefill[i] < self.kv_need[i]:
                if not chunked:
                    continue
                chunk = min(int(self.kv_need[i] - self.prefill[i]), budget)
                if chunk > 0:
                    members.append((i, chunk))
                    budget -= chunk
                continue
            if returned[i] and i not in grown:
                continue
            if budget >= 1:
                members.append((i, 1))
                budget -= 1
        for i in self._fcfs(waiting):
            chunk = int(self.kv_need[i] - self.prefill[i])
            alloc = ((int(self.kv_need[i]) + 1 + step - 1) // step) * step
            cost = self._fp(alloc)
            if cost > free:
                break
            if chunk > 0:
                if chunked:
                    chunk = min(chunk, budget)
                    if chunk < 1:
                        break
                elif budget < chunk:
                    break
                members.append((i, chunk))
                budget -= chunk
            actions.append(("allocate", i, alloc, 0, -1, 0))
            free -= cost
        return self._plan_dict(members, preempt, actions)

    def _plan_evict_returned(self, strat, order, demand):
        """scheduler.py:841-936 shared shape of rlp / s3: returned requests
        evict themselves, decodes join, then admissions in `order` until the
        first that does not fit."""
        sc = self.cfg.sched
        running, waiting, eff, ready = self._baseline_views()
        running = [i for i in running if ready[i]]
        free = self.free_tokens()
        budget = sc.token_budget
        members, actions = [], []
        preempt = [(i, strat) for i in running if eff[i] < int(self.used[i]) + 1]
        removed = {i for i, _ in preempt}
        for i in running:
            if i in removed or self.state[i] != RUNNING or self.prefill[i] < self.kv_need[i]:
                continue
            if budget >= 1:
                members.append((i, 1))
                budget -= 1
        for i in order([i for i in waiting if ready[i]]):
            chunk = int(self.kv_need[i] - self.prefill[i])
            alloc = demand(i, eff[i])
            cost = self._cost(i, alloc)
            if cost > free:
                break
            if chunk > 0:
                if budget < chunk:
                    break
                members.append((i, chunk))
                budget -= chunk
            actions.append(("grow" if self.holds[i] else "allocate", i, alloc, 0, -1, 0))
            free -= cost
        return self._plan_dict(members, preempt, actions)

    def plan_rlp(self):
        """scheduler.py:841-890: shortest predicted remaining bucket first."""
        pad = self.cfg.sched.rlp_padding

        def rem(i):
            return max(1, int(self.pred[i] - self.gen[i]))

        def order(w):
            return sorted(w, key=lambda i: (rem(i) // 50, int(self.arr[i]), self.rid[i]))
        return self._plan_evict_returned(RECOMPUTE, order,
                                         lambda i, e: int(self.kv_need[i]) + rem(i) + pad - e)

    def plan_s3(self):
        """scheduler.py:893-936: FCFS, bucketed output demand doubling per preemption."""
        bt = self.cfg.sched.s3_bucket_tokens

        def demand(i, e):
            out = max(1, -(-max(1, int(self.pred[i])) // bt)) * bt * (2 ** int(self.pcount[i]))
            return max(0, int(self.kv_need[i]) + out - e)
        return self._plan_evict_returned(SWAP, self._fcfs, demand)

    def plan(self):
        pol = self.cfg.sched.policy
        if pol == "vllm_block":
            return self.plan_vllm_block(False)
        if pol == "sarathi_chunked":
            return self.plan_vllm_block(True)
        if pol == "rlp":
            return self.plan_rlp()
        if pol == "s3":
            return self.plan_s3()
        return self.plan_cacheopt()

    def plan_cacheopt(self):
        """scheduler.py:408-753.  The pool is not mutated while planning, so
        snapshot quantities (engine.py:284-317) are read straight from it."""
        cfg = self.cfg
        sc = cfg.sched
        B = sc.small_block_b
        eps = sc.epsilon_us
        bs = self.bs
        now = self.now
        live = np.nonzero((self.state >= WAITING) & (self.state <= PREEMPTED))[0]
        st = self.state[live]
        no_first = self.first_tok[live] < 0
        rt_arr = np.where(no_first, self.slo_ttft[live] - (now - self.arr[live]),
                          self.slo_tbt[live] - (now - self.last_tok[live]))
        wait_mask = (st == WAITING) | (st == PREEMPTED)
        run_mask = st == RUNNING
        ids_np = self._ids_np
        # classify_critical over waiting views, all of which are ready
        # (scheduler.py:129-141, engine.py:311-312)
        crit_w = wait_mask & (rt_arr >= -eps) & (rt_arr - self.t_i < eps)
        wl = live[crit_w]
        o = np.lexsort((ids_np[wl], rt_arr[crit_w]))
        n_w = [int(x) for x in wl[o]]
        pm = wait_mask & ~crit_w
        pl = live[pm]
        prt = rt_arr[pm]
        blown = prt < 0
        qv = np.where(blown, self.arr[pl], prt)
        o = np.lexsort((ids_np[pl], qv, blown))          # queue_key, scheduler.py:151-157
        n_wp_arr = pl[o]
        running_all = [int(x) for x in live[run_mask]]   # arrival order (engine.py:321-323)
        eff_cache = {}

        def eff_of(i):
            v = eff_cache.get(i)
            if v is None:
                v = eff_cache[i] = self.eff_alloc(i)
            return v

        class _Lazy(dict):
            def __missing__(d, i):
                return eff_of(i)

        class _LazyRt(dict):
            def __missing__(d, i):
                v = d[i] = self._rt(i)
                return v

        eff = _Lazy()
        rt = _LazyRt()

        used = self.used
        kvn = self.kv_need
        pdone = self.prefill
        est = self.est
        gen = self.gen

        def est_rem(i):
            return max(0, int(est[i] - gen[i]))

        def target(i):
            return max(int(used[i]), int(kvn[i])) + est_rem(i)

        def is_guest(i):
            return bool(self.holds[i]) and self.host[i] >= 0

        def returned(i):
            return self.state[i] == RUNNING and eff[i] < int(used[i]) + 1

        def ready(i):
            return self.state[i] != RUNNING or now >= self.ready_at[i]

        def held(i):
            return int(self.granted[i]) if self.holds[i] else 0

        def cost_of(i, grant):
            """scheduler.py:350-354."""
            if is_guest(i):
                return 0
            h = held(i)
            return self._fp(h + grant) - self._fp(h)

        def qkey(i):
            r = rt[i]
            return (1, int(self.arr[i]), self.rid[i]) if r < 0 else (0, r, self.rid[i])

        # returned running, ready (scheduler.py:142-150)
        n_r, n_rp = [], []
        for i in running_all:
            if not ready(i) or not returned(i):
                continue
            r = rt[i]
            if r >= -eps and r - self.t_i < eps:
                n_r.append(i)
            else:
                n_rp.append(i)
        n_r.sort(key=lambda i: (rt[i], self.rid[i]))
        n_rp.sort(key=qkey)

        free = self.free_tokens()
        rsv_blocks = self.rsv_cur
        members: List[Tuple[int, int]] = []
        preempt: List[Tuple[int, int]] = []
        actions: List[tuple] = []   # (kind, idx, tokens, blocks, host, start)
        claims: List[Tuple[int, int]] = []
        deferred: List[int] = []
        granted_members: List[Tuple[int, int]] = []
        embedded = set()
        removed = set()

        # embedding hosts: decode-phase non-guest holders (scheduler.py:425-430)
        triples = [(i, int(self.granted[i]), int(used[i])) for i in running_all
                   if not is_guest(i) and self.holds[i] and pdone[i] >= kvn[i]]

        def try_embed(i):
            """scheduler.py:432-449."""
            if eff[i] > 0 or self.pcount[i] > 0:
                return False
            out = max(est_rem(i), int(self.pred[i] - gen[i]), 1)
            q = self.find_host([t for t in triples if t[0] not in removed], int(kvn[i]), out)
            if q is None:
                return False
            actions.append(("embed", i, int(kvn[i]) + out, 0, q[0], q[1]))
            embedded.add(i)
            triples[:] = [t for t in triples if t[0] != q[0]]
            return True

        pending_nw = []
        for i in n_w:
            if try_embed(i):
                granted_members.append((i, int(kvn[i] - pdone[i])))
            else:
                pending_nw.append(i)

        def nw_need(i):
            return max(0, int(kvn[i]) + B - eff[i])

        demand = sum(cost_of(i, nw_need(i)) for i in pending_nw)
        demand += sum(cost_of(i, B) for i in n_r if not is_guest(i))
        shortfall = max(0, demand - free)
        if shortfall > 0:
            shortfall -= min(shortfall, rsv_blocks * bs)
        if shortfall > 0:
            crit = set(pending_nw) | set(n_r)
            cands = [i for i in running_all if not is_guest(i) and i not in crit
                     and self.holds[i] and self.release_gain(i) > 0]
            slo_rule = sc.victim_rule == "slo"
            if slo_rule:
                cands = [i for i in cands if pdone[i] >= kvn[i]]
                edges = sc.buckets.slo_edges_us
                step_tok = sc.buckets.token_step

                def vkey(i):  # preemption.py:46-64
                    sb = sum(1 for e in edges if self.slo_tbt[i] >= e)
                    return (-sb, -(est_rem(i) // step_tok), int(used[i]), self.rid[i])
            else:
                def vkey(i):  # scheduler.py:397-398
                    return (-int(self.arr[i]), self.rid[i])
            queued = int(np.count_nonzero(wait_mask))
            tr = cfg.truth
            for i in sorted(cands, key=vkey):
                if shortfall <= 0:
                    break
                strat = self._strategy(i)
                if slo_rule:
                    s = max(1, int(used[i]))  # scheduler.py:362-375
                    ms = swap_ms(tr.swap_true, s) if strat == SWAP else recompute_ms(tr.recompute_true, s)
                    charge = int(ms * 1000 + 0.5) + self.t_i * (1 + queued)
                    if not rt[i] > charge:
                        continue
                gain = self.release_gain(i)
                preempt.append((i, strat))
                removed.add(i)
                free += gain
                shortfall -= gain
            if shortfall > 0:
                for i in sorted(pending_nw, key=lambda i: (-rt[i], self.rid[i])):
                    if shortfall <= 0:
                        break
                    shortfall -= cost_of(i, nw_need(i))
                    pending_nw.remove(i)
                    deferred.append(i)

        running = [i for i in running_all if i not in removed]

        # N_r continuation (scheduler.py:515-532)
        stalled = set()
        for i in n_r:
            if i in removed:
                continue
            c = cost_of(i, B)
            if is_guest(i):
                actions.append(("grow", i, B, 0, -1, 0))
            elif c <= free:
                actions.append(("grow", i, B, 0, -1, 0))
                free -= c
            else:
                nb = (B + bs - 1) // bs
                if rsv_blocks >= nb:
                    actions.append(("reserve", i, 0, nb, -1, 0))
                    rsv_blocks -= nb
                else:
                    stalled.add(i)
        # N'_r resumption (scheduler.py:537-550)
        resumed = set()
        for i in n_rp:
            if i in removed:
                continue
            if is_guest(i):
                actions.append(("grow", i, B, 0, -1, 0))
                resumed.add(i)
                continue
            c = cost_of(i, B)
            if c <= free:
                actions.append(("grow", i, B, 0, -1, 0))
                free -= c
                resumed.add(i)
        # critical admissions (scheduler.py:553-574)
        for i in pending_nw:
            need = nw_need(i)
            c = cost_of(i, need)
            if c <= free:
                actions.append(("grow" if self.holds[i] else "allocate", i, need, 0, -1, 0))
                free -= c
            elif not is_guest(i):
                nb = (need + bs - 1) // bs
                if nb <= rsv_blocks:
                    actions.append(("reserve", i, 0, nb, -1, 0))
                    rsv_blocks -= nb
                else:
                    deferred.append(i)
                    continue
            else:
                deferred.append(i)
                continue
            chunk = int(kvn[i] - pdone[i])
            if chunk > 0:
                granted_members.append((i, chunk))

        # decode members (scheduler.py:576-590)
        n_r_set = set(n_r)
        decode = 0
        for i in running:
            if not ready(i) or pdone[i] < kvn[i]:
                continue
            if returned(i):
                if i in stalled:
                    continue
                if i not in n_r_set and i not in resumed:
                    continue
            members.append((i, 1))
            decode += 1
        members.extend(granted_members)
        consumed = decode + sum(t for _, t in granted_members)

        # token budget fill (scheduler.py:182-200, 596-598)
        budget = sc.token_budget
        if len(n_wp_arr):
            chunks = (kvn[n_wp_arr] - pdone[n_wp_arr])
            over = np.nonzero(consumed + np.cumsum(chunks) > budget)[0]
            k = int(over[0]) if len(over) else len(n_wp_arr)
        else:
            k = 0
        selected = [int(x) for x in n_wp_arr[:k]]
        overflow = consumed > budget

        # participants (scheduler.py:600-638)
        parts: List[Tuple[int, int]] = []
        in_parts = set()
        member_ready: List[int] = []
        for i in selected:
            if try_embed(i):
                member_ready.append(i)
                continue
            need = max(target(i), int(kvn[i]) + 1) - eff[i]
            if need <= 0:
                member_ready.append(i)
            else:
                parts.append((i, need))
                in_parts.add(i)
        for i in n_rp:
            if i in removed or is_guest(i) or i not in resumed:
                continue
            res = max(0, target(i) - eff[i] - B)
            if res > 0:
                parts.append((i, res))
                in_parts.add(i)
        m = sc.preallocate_m
        pro = [i for i in running if not returned(i) and eff[i] < target(i) and est_rem(i) <= m]
        pro.sort(key=lambda i: (est_rem(i), self.rid[i]))
        for i in pro:
            if i in removed or is_guest(i) or i in in_parts:
                continue
            parts.append((i, target(i) - eff[i]))
            in_parts.add(i)
        for i in running:
            if is_guest(i) or not ready(i) or pdone[i] < kvn[i] or returned(i):
                continue
            if eff[i] - int(used[i]) > m or i in in_parts:
                continue
            parts.append((i, max(target(i), int(used[i]) + 1 + B) - eff[i]))
            in_parts.add(i)

        # amortized round (scheduler.py:640-682)
        def amortize(ps, supply):
            dem = [(self.rid[i], mt, max(1, rt[i]), max(1, int(kvn[i]))) for i, mt in ps]
            g = (split_largest_remainder_inverted if sc.invert_amortization else split_largest_remainder)(dem, supply)
            total = sum(d[1] for d in dem)
            if total > supply and g:
                fl = {r: (x // bs) * bs for r, x in g.items()}
                left = (supply - sum(fl.values())) // bs
                for r in sorted(g, key=lambda r: (-(g[r] - fl[r]), r))[:left]:
                    fl[r] += bs
                g = fl
            return g, total

        n_dec = sum(1 for i in running if not is_guest(i) and pdone[i] >= kvn[i])
        runway = sc.decode_runway_iters * n_dec
        inflight = [(i, mt) for i, mt in parts if self.state[i] == RUNNING]
        admitting = [(i, mt) for i, mt in parts if self.state[i] != RUNNING]
        flight_supply = (free // bs) * bs
        grants, flight_total = amortize(inflight, flight_supply)
        spent = sum(grants.values())
        admit_supply = (max(0, free - spent - runway) // bs) * bs
        ag, admit_total = amortize(admitting, admit_supply)
        grants.update(ag)
        sated = flight_total <= flight_supply and admit_total <= admit_supply

        fulfilled = [i for i in running if not is_guest(i) and not returned(i) and eff[i] >= target(i)]
        claimed = set()
        for i, need in parts:
            g = grants.get(self.rid[i], 0)
            if self.state[i] != RUNNING:
                if eff[i] + g < int(kvn[i]) + 1:
                    continue
                actions.append(("grow" if self.holds[i] else "allocate", i, g, 0, -1, 0))
                free -= cost_of(i, g)
                member_ready.append(i)
            elif g > 0:
                actions.append(("grow", i, g, 0, -1, 0))
                free -= cost_of(i, g)
                if returned(i) and eff[i] + g >= int(used[i]) + 1:
                    members.append((i, 1))
            if g < need:
                # NB: rebinds the decode runway used by the extras gate below
                # (scheduler.py:710 shadows :671)
                runway = eff[i] + g - int(used[i])
                resid = need - g
                lim = max(0, runway)
                best = None
                for p in fulfilled:
                    if p in claimed:
                        continue
                    er = est_rem(p)
                    if er > lim or self.release_gain(p) < resid:
                        continue
                    key = (er, self.rid[p])
                    if best is None or key < best[0]:
                        best = (key, p)
                if best is not None:
                    claims.append((i, best[1]))
                    claimed.add(best[1])
        for i in member_ready:
            if self.state[i] == WAITING:
                members.append((i, int(kvn[i] - pdone[i])))

        # case 2 extras (scheduler.py:726-748)
        if sated:
            floors = [int(self.slo_tbt[x]) for x in running
                      if self.last_tok[x] >= 0 and not returned(x)
                      and not self.max_tbt[x] > self.slo_tbt[x]
                      and int(self.slo_tbt[x]) - (now - int(self.last_tok[x])) >= 0]
            tbt_floor = min(floors) if floors else None
            batch_now = sum(t for _, t in members)
            cand = n_wp_arr[k:]
            if len(cand):
                # vectorised walk: skip while need == 0 or cost > free - runway,
                # stop at the latency gate (free only decreases, so a skipped
                # item stays skipped)
                hold = self.holds[cand]
                g0 = np.where(hold, self.granted[cand], 0)
                effc = g0.copy()
                if self.guests:
                    for x in np.nonzero(np.isin(cand, list(self.guests)))[0]:
                        effc[x] = self.eff_alloc(int(cand[x]))
                tg = np.maximum(used[cand], kvn[cand]) + np.maximum(0, est[cand] - gen[cand])
                needs = np.maximum(0, tg - effc)
                guest = hold & (self.host[cand] >= 0)
                costs = np.where(guest, 0, ((g0 + needs + bs - 1) // bs) * bs - ((g0 + bs - 1) // bs) * bs)
                # cand = N'_w after the selected prefix; embedded requests come
                # from N_w or the prefix, so cand is exactly the extras list
                ok = needs > 0
                pos = 0
                while True:
                    feas = np.nonzero(ok[pos:] & (costs[pos:] <= free - runway))[0]
                    if not len(feas):
                        break
                    x = pos + int(feas[0])
                    i = int(cand[x])
                    if tbt_floor is not None:
                        if iter_ms(cfg, batch_now + int(kvn[i])) * 1000 > tbt_floor:
                            break
                    actions.append(("grow" if self.holds[i] else "allocate", i, int(needs[x]), 0, -1, 0))
                    free -= int(costs[x])
                    pos = x + 1
        if getattr(self, "debug_sizes", None) is not None:  # development aid: per-step set sizes
            self.debug_sizes.append(dict(
                running=len(running_all), n_w=len(n_w), n_r=len(n_r), n_rp=len(n_rp), triples=len(triples),
                n_wp=len(n_wp_arr), pending=len(pending_nw), victims=len(preempt), deferred=len(deferred),
                selected=len(selected), parts=len(parts), pro=len(pro), fulfilled=len(fulfilled), sated=sated,
                claims=len(claims), actions=len(actions), members=len(members), granted_members=len(granted_members)))
        return dict(members=members, preempt=preempt, actions=actions, claims=claims,
                    deferred=deferred, overflow=overflow or sum(t for _, t in members) > budget,
                    batch_tokens=sum(t for _, t in members))

    # -- apply (engine.py:437-536) ------------------------------------------

    def _apply(self, plan):
        now = self.now
        for i, s in plan["preempt"]:
            self._preempt(i, s, now)
        failed = set()
        acted = []
        live_states = (WAITING, RUNNING, PREEMPTED)
        for kind, i, tok, nb, h, start in plan["actions"]:
            if i in failed or self.state[i] not in live_states:
                continue
            if kind == "allocate":
                ok = self.pool_allocate(i, tok)
            elif kind == "grow":
                ok = self.pool_grow(i, tok)
            elif kind == "reserve":
                ok = self.pool_draw_reserved(i, nb)
            else:
                ok = self.pool_embed(i, tok, h, start)
            if ok:
                acted.append(i)
                self.alloc_kvc[i] = self.granted[i]
                continue
            if kind == "grow" and self.holds[i] and self.host[i] >= 0 and self.state[i] == RUNNING:
                if self.pool_promote(i):
                    if self.pool_grow(i, tok):
                        acted.append(i)
                        self.alloc_kvc[i] = self.granted[i]
                        continue
                    failed.add(i)
                    continue
                self._preempt(i, self._strategy(i), now, cause="squeeze")
            failed.add(i)
        for i in dict.fromkeys(acted):
            if self.state[i] == PREEMPTED:
                self._readmit(i)
        out = []
        batch = 0
        seen = set()
        for i, tok in plan["members"]:
            if i in failed or i in seen:
                continue
            seen.add(i)
            s = self.state[i]
            if s not in live_states:
                continue
            if s == WAITING:
                if not self.holds[i] or self.granted[i] < self.prefill[i] + tok:
                    continue
                self.state[i] = RUNNING
                if self.first_start[i] < 0:
                    self.first_start[i] = now
                    self._ev(ev="admit", t=now, req=self.rid[i])
            elif s != RUNNING:
                continue
            if self.ready_at[i] > now:
                continue
            if self.prefill[i] >= self.kv_need[i]:
                if self.eff_alloc(i) < self.used[i] + 1:
                    continue
            elif self.granted[i] < self.prefill[i] + tok:
                continue
            out.append((i, tok))
            batch += tok
        for w, p in plan["claims"]:
            if self.state[w] in live_states and self.state[p] in live_states:
                self.claims.setdefault(p, w)
        return out, batch

    # -- emission (engine.py:540-591) ----------------------------------------

    def _token(self, i, t):
        self.gen[i] += 1
        self.gen_total += 1
        if self.first_tok[i] < 0:
            self.first_tok[i] = t
        else:
            self.max_tbt[i] = max(int(self.max_tbt[i]), t - int(self.last_tok[i]))
        self.last_tok[i] = t
        self.token_times[i].append(t)

    def _emit(self, members, t):
        done = []
        for i, tok in members:
            if self.prefill[i] < self.kv_need[i]:
                self.prefill[i] += tok
                self.set_used(i, int(self.prefill[i]))
                if self.prefill[i] >= self.kv_need[i] and self.gen[i] == 0:
                    self._token(i, t)
            else:
                self.set_used(i, int(self.used[i]) + 1)
                self._token(i, t)
            if self.gen[i] >= self.tout[i]:
                done.append(i)
        for i in done:
            self._complete(i, t)

    def _collisions(self, now):
        """engine.py:573-591; hosts visited in record-creation order."""
        hosts = sorted((h for h, gl in self.guests.items() if gl), key=lambda h: self.rec_seq[h])
        for h in hosts:
            if not self.holds[h] or self.state[h] != RUNNING:
                continue
            gl = list(self.guests.get(h, []))
            if not gl:
                continue
            u = int(self.used[h])
            for g in sorted(gl, key=lambda g: self.off[g]):
                if u >= self.off[g]:
                    if self.pool_promote(g):
                        continue
                    if self.state[g] == RUNNING:
                        self._preempt(g, self._strategy(g), now, cause="collision")

    def _next_event(self):
        """engine.py:593-602."""
        c = []
        if self.next_pending < self.n:
            c.append(int(self.arr[self.next_pending]))
        r = np.nonzero((self.state == RUNNING) & (self.ready_at > self.now))[0]
        if len(r):
            c.append(int(self.ready_at[r].min()))
        return min(c) if c else None

    # -- main loop (engine.py:606-672) ----------------------------------------

    def step(self) -> bool:
        if self.n_live == 0 and self.next_pending >= self.n:
            return False
        if self.now > self.horizon:
            return False
        if self.n_live == 0:
            self.now = max(self.now, int(self.arr[self.next_pending]))
        self._admit_arrivals()
        plan = self.plan()
        self.last_plan = plan
        members, batch = self._apply(plan)
        if not members and not plan["actions"] and not plan["preempt"]:
            nxt = self._next_event()
            if nxt is None:
                self.stalled = True
                return False
            self.now = nxt
            return True
        il = to_us(iter_ms(self.cfg, batch))
        end = self.now + il
        self.t_i = il
        self._ev(ev="iter", t=self.now, end=end, tokens=batch,
                 members=[[self.rid[i], t] for i, t in members])
        self._emit(members, end)
        self._collisions(end)
        self.samples.append((self.fp_sum, self.used_sum))
        self.iters += 1
        ve = self.cfg.validate_every
        if ve and self.iters % ve == 0:
            self.check_invariants()
        self.now = end
        return True

    def run(self, max_steps: Optional[int] = None) -> int:
        """engine.py:643-661 loop (metrics are computed by the caller)."""
        streak = 0
        last = None
        steps = 0
        while max_steps is None or steps < max_steps:
            mark = (self.now, self.gen_total, self.n_live, self.n - self.next_pending, self.fp_sum)
            if mark == last:
                streak += 1
                if streak > NO_PROGRESS_LIMIT:
                    raise RuntimeError(f"no progress after {streak} rounds at t={self.now}")
            else:
                streak = 0
            last = mark
            steps += 1
            if not self.step():
                break
        return steps

    # -- read-outs ----------------------------------------------------------

    def metrics(self) -> dict:
        """engine.py:132-211 compute_metrics (+ :662-671 makespan) over the
        final state, as MetricsReport.to_dict(): requests visited in the
        caller's order (the reference's dict order), numpy percentile/mean."""
        def pct(vals):
            if len(vals) == 0:
                return {"p50": 0.0, "p90": 0.0, "p99": 0.0, "max": 0.0, "mean": 0.0}
            a = np.asarray(vals, dtype=float)
            return {"p50": float(np.percentile(a, 50)), "p90": float(np.percentile(a, 90)),
                    "p99": float(np.percentile(a, 99)), "max": float(a.max()), "mean": float(a.mean())}

        def mean(xs):
            return float(np.mean(xs)) if xs else 0.0

        n = self.n
        ttfts, gaps_all, norm, waits, execs, pdec = [], [], [], [], [], []
        ok_ttft = ok_tbt = done = 0
        for i in self.input_order:
            tt = self.token_times[i]
            gaps = [b - a for a, b in zip(tt, tt[1:])]
            arr = int(self.arr[i])
            if self.first_tok[i] >= 0 and int(self.first_tok[i]) - arr <= int(self.slo_ttft[i]):
                ok_ttft += 1
            if self.state[i] != COMPLETED:
                continue
            done += 1
            if all(g <= int(self.slo_tbt[i]) for g in gaps):
                ok_tbt += 1
            ttfts.append(int(self.first_tok[i]) - arr)
            gaps_all.extend(gaps)
            norm.append((int(self.completion[i]) - arr) / int(self.tout[i]))
            waits.append(int(self.first_start[i]) - arr)
            pdec.append(int(self.ptime[i]))
            execs.append(int(self.completion[i]) - int(self.first_start[i]) - int(self.ptime[i]))
        hit = [i for i in self.input_order if self.pcount[i] > 0]
        makespan = max(0, self.now - self.first_arrival)
        span_s = makespan / 1_000_000 if makespan > 0 else 0.0
        cap = self.capacity
        if self.samples:
            util = float(np.mean([fp / cap for fp, _ in self.samples]))
            frag = float(np.mean([(fp - u) / cap for fp, u in self.samples]))
        else:
            util = frag = 0.0
        return dict(
            policy=self.cfg.sched.policy, seed=self.cfg.seed, num_requests=n, completed=done,
            makespan_us=makespan, ttft_us=pct(ttfts), tbt_us=pct(gaps_all),
            ttft_attainment=ok_ttft / n if n else 0.0, tbt_attainment=ok_tbt / n if n else 0.0,
            normalized_us_per_token=pct(norm), preemption_total=int(self.pcount.sum()),
            preempted_requests=len(hit), preemption_time_us=pct([int(self.ptime[i]) for i in hit]),
            throughput_rps=done / span_s if span_s else 0.0,
            throughput_tps=int(self.gen.sum()) / span_s if span_s else 0.0,
            kvc_utilization_mean=util, kvc_fragmentation_mean=frag,
            waiting_us_mean=mean(waits), execution_us_mean=mean(execs), preemption_us_mean=mean(pdec),
        )

    def final_state(self) -> Dict[str, np.ndarray]:
        """Per-request outcome arrays in arrival order, for parity checks."""
        return dict(
            req_id=np.array(self.rid, dtype=np.int64),
            state=self.state.astype(np.int64), generated=self.gen.copy(),
            used=self.used.copy(), kv_need=self.kv_need.copy(),
            prefill_done=self.prefill.copy(), preemption_count=self.pcount.copy(),
            preemption_time_us=self.ptime.copy(), first_token_at_us=self.first_tok.copy(),
            last_token_at_us=self.last_tok.copy(), max_tbt_us=self.max_tbt.copy(),
            ready_at_us=self.ready_at.copy(), first_start_us=self.first_start.copy(),
            completion_us=self.completion.copy(), allocated_kvc=self.alloc_kvc.copy(),
            predicted=self.pred.copy(), estimated=self.est.copy(),
            holds=self.holds.astype(np.int64), granted=np.where(self.holds, self.granted, 0),
        )
