"""Host-side preparation of one engine instance: everything the reference
derives from floating point or from numpy's RNG is evaluated HERE, once, with
Python's own IEEE-double semantics, and handed to the device as integers:

- the run's confidence and padding (engine.py:256-266, estimation.py:102-119)
- the sweet spot s* (scheduler.py:378-393, preemption.py:176-195)
- per-length swap / recompute charge LUTs (engine.py:372, 392-397;
  scheduler.py:368-374)
- ``noise_draws``: the host twin of the predictor noise draws (consumed from
  default_rng([seed, 3]) in (arrival, id) order exactly as engine.py:267/344-351
  consumes it); the engine itself draws them on the GPU (devrng.py), this one
  is the bench's host-side comparison.

The device never evaluates a transcendental; the only float expression it
evaluates is the iteration latency (costmodel.py:51-55), with explicit
round-to-nearest double intrinsics.
"""
from __future__ import annotations

import math
from typing import Tuple

import numpy as np

from .config import EngineConfig, RecomputeModel, SwapModel


def run_confidence(cfg: EngineConfig, arrivals_sorted: np.ndarray) -> float:
    if cfg.fixed_confidence is not None:
        return cfg.fixed_confidence
    n = len(arrivals_sorted)
    rate = 0.0
    if n:
        span = int(arrivals_sorted[-1]) - int(arrivals_sorted[0])
        if span > 0:
            rate = (n - 1) / (span / 1_000_000)
    pol = cfg.confidence
    if rate < 0:
        raise ValueError("arrival_rate must be >= 0")
    raw = pol.alpha / (1.0 + pol.beta * rate)
    return min(pol.clamp_hi, max(pol.clamp_lo, raw))


def run_padding(cfg: EngineConfig, confidence: float) -> int:
    pc = cfg.predictor
    if pc.fixed_padding is not None:
        return pc.fixed_padding
    width = pc.bin_width - 1  # hi - lo of the enclosing bin
    if not 0.0 < confidence < 1.0:
        raise ValueError("confidence must be in (0, 1)")
    bound = width * math.sqrt(-math.log(1.0 - confidence) / 2.0)
    return min(width, math.floor(bound + 0.5))


def sweet_spot(swp: SwapModel, rec: RecomputeModel, s_max: int = 1_000_000) -> int:
    """Largest S with L_r(S) <= L_s(S) by integer bisection; one model
    dominating everywhere encodes as all-swap (0) / all-recompute (2**62)."""
    def gap(s):
        return rec.predict(s) - swp.predict(s)
    lo, hi = 1, s_max
    if gap(lo) > 0 or gap(hi) <= 0:
        return 0 if rec.predict(1) > swp.predict(1) else (1 << 62)
    while hi - lo > 1:
        mid = (lo + hi) // 2
        lo, hi = (mid, hi) if gap(mid) <= 0 else (lo, mid)
    return lo


def charge_luts(cfg: EngineConfig, s_max: int) -> Tuple[np.ndarray, ...]:
    """Integer charges indexed by sequence length S (index 0 unused)."""
    swp, rec = cfg.truth.swap_true, cfg.truth.recompute_true
    swap_half = np.zeros(s_max + 1, dtype=np.int64)
    rec_us = np.zeros(s_max + 1, dtype=np.int64)
    surv_swap = np.zeros(s_max + 1, dtype=np.int64)
    surv_rec = np.zeros(s_max + 1, dtype=np.int64)
    for s in range(1, s_max + 1):
        ls = swp.predict(s)
        lr = rec.predict(s)
        swap_half[s] = math.floor((ls / 2.0) * 1000 + 0.5)
        rec_us[s] = math.floor(lr * 1000 + 0.5)
        surv_swap[s] = int(ls * 1000 + 0.5)
        surv_rec[s] = int(lr * 1000 + 0.5)
    return swap_half, rec_us, surv_swap, surv_rec


def noise_draws(cfg: EngineConfig, n: int) -> Tuple[np.ndarray, np.ndarray]:
    """Predictor error and direction-flip draws for n arrivals, in the order
    the engine admits them."""
    pc = cfg.predictor
    err = np.zeros(n, dtype=np.int32)
    flip = np.zeros(n, dtype=np.uint8)
    need_flip = pc.direction_accuracy < 1.0
    if pc.error_dist == "zero" and not need_flip:
        return err, flip
    rng = np.random.default_rng([cfg.seed, 3])
    s = int(pc.error_scale)
    miss = 1.0 - pc.direction_accuracy
    for k in range(n):
        if pc.error_dist == "uniform":
            if s > 0:
                err[k] = int(rng.integers(-s, s + 1))
        elif pc.error_dist == "normal":
            err[k] = math.floor(float(rng.normal(0.0, pc.error_scale)) + 0.5)
        if need_flip:
            flip[k] = 1 if rng.random() < miss else 0
    return err, flip


def iteration_us(cfg: EngineConfig, batch_tokens: int) -> int:
    c = cfg.iter_cost
    return math.floor((c.base_ms + c.per_token_ms * batch_tokens) * 1000 + 0.5)


def bin_of(predicted: int, width: int) -> Tuple[int, int]:
    k = (predicted + width - 1) // width
    return (k - 1) * width + 1, k * width
