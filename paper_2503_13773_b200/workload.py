"""Synthetic trace input (host side, not part of the device path).

Produces the same traces as the reference's workload module
(workload.py:85-109 generate, :181-194 assign_slos) for the same seeds, so a
trace built here and one built by the reference are interchangeable.  The
dataset presets are the Table-1 statistics of the paper (workload.py:60-76).
"""
from __future__ import annotations

import csv
import dataclasses
import math
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence

import numpy as np

from .core import US_PER_S, Request

HOUR_US = 3_600 * US_PER_S  # placeholder SLO until assign_slos runs


@dataclass(frozen=True)
class TraceSpec:
    arrival_rate: float
    num_requests: int
    input_mean: float
    input_min: int
    input_max: int
    output_mean: float
    output_min: int
    output_max: int
    length_cv: float = 1.0

    def __post_init__(self) -> None:
        if self.arrival_rate <= 0:
            raise ValueError("arrival_rate must be > 0")
        if self.num_requests < 1:
            raise ValueError("num_requests must be >= 1")
        for side in ("input", "output"):
            lo, hi = getattr(self, side + "_min"), getattr(self, side + "_max")
            if not 1 <= lo <= hi:
                raise ValueError(f"{side} bounds must satisfy 1 <= min <= max")
            if not lo <= getattr(self, side + "_mean") <= hi:
                raise ValueError(f"{side}_mean must lie within its bounds")
        if self.length_cv <= 0:
            raise ValueError("length_cv must be > 0")

    def sized(self, num_requests: int, arrival_rate: Optional[float] = None) -> "TraceSpec":
        rate = self.arrival_rate if arrival_rate is None else arrival_rate
        return dataclasses.replace(self, num_requests=num_requests, arrival_rate=rate)


PRESETS: Dict[str, TraceSpec] = {
    name: TraceSpec(rate, 1000, im, ilo, ihi, om, olo, ohi)
    for name, rate, im, ilo, ihi, om, olo, ohi in (
        ("alpaca", 32.0, 19.31, 9, 2470, 58.41, 13, 292),
        ("sharegpt", 28.0, 161.31, 16, 3200, 337.99, 19, 991),
        ("bookcorpus", 1.2, 1952.11, 18, 8192, 681.2, 32, 1041),
    )
}


def _lognormal(mean: float, cv: float):
    s2 = math.log(1.0 + cv * cv)
    return math.log(mean) - s2 / 2.0, math.sqrt(s2)


def trace_arrays(spec: TraceSpec, seed: int) -> Dict[str, np.ndarray]:
    """Columnar trace: arrival_us, prompt_len, true_output_len (int64)."""
    n = spec.num_requests
    gaps = np.random.default_rng([seed, 0]).exponential(1.0 / spec.arrival_rate, size=n)
    arrival = np.floor(np.cumsum(gaps) * US_PER_S + 0.5).astype(np.int64)
    mu, sig = _lognormal(spec.input_mean, spec.length_cv)
    prompt = np.rint(np.random.default_rng([seed, 1]).lognormal(mu, sig, size=n))
    mu, sig = _lognormal(spec.output_mean, spec.length_cv)
    out = np.rint(np.random.default_rng([seed, 2]).lognormal(mu, sig, size=n))
    return {
        "arrival_us": arrival,
        "prompt_len": np.clip(prompt, spec.input_min, spec.input_max).astype(np.int64),
        "true_output_len": np.clip(out, spec.output_min, spec.output_max).astype(np.int64),
    }


def generate(spec: TraceSpec, seed: int) -> List[Request]:
    cols = trace_arrays(spec, seed)
    return [Request(id=i, arrival_us=int(a), prompt_len=int(p), true_output_len=int(o),
                    slo_ttft_us=HOUR_US, slo_tbt_us=HOUR_US)
            for i, (a, p, o) in enumerate(zip(cols["arrival_us"], cols["prompt_len"],
                                              cols["true_output_len"]))]


def ingest_csv(path: str) -> List[Request]:
    """CSV with header arrival_us,prompt_len,output_len (non-decreasing
    arrivals); errors name the 1-based line."""
    header = ["arrival_us", "prompt_len", "output_len"]
    out: List[Request] = []
    with open(path, newline="") as fh:
        rows = csv.reader(fh)
        first = next(rows, None)
        if first is None:
            raise ValueError(f"{path}: empty file")
        if [h.strip() for h in first] != header:
            raise ValueError(f"{path}: bad header {first!r}, expected {','.join(header)}")
        last = -1
        for line, row in enumerate(rows, start=2):
            if not row:
                continue
            if len(row) != 3:
                raise ValueError(f"{path} line {line}: expected 3 fields")
            try:
                a, p, o = (int(x) for x in row)
            except ValueError:
                raise ValueError(f"{path} line {line}: non-integer field in {row!r}") from None
            if a < last:
                raise ValueError(f"{path} line {line}: arrival {a} before previous {last}")
            last = a
            try:
                out.append(Request(len(out), a, p, o, HOUR_US, HOUR_US))
            except ValueError as exc:
                raise ValueError(f"{path} line {line}: {exc}") from None
    return out


@dataclass(frozen=True)
class SloPolicy:
    scale_lo: float = 0.5
    scale_hi: float = 2.5
    chunk_budget: int = 2048

    def __post_init__(self) -> None:
        if not 0 < self.scale_lo <= self.scale_hi:
            raise ValueError("need 0 < scale_lo <= scale_hi")
        if self.chunk_budget < 1:
            raise ValueError("chunk_budget must be >= 1")

    def chunk_factor(self, prompt_len: int) -> int:
        return max(1, math.ceil(prompt_len / self.chunk_budget))


def slo_arrays(prompt_len: np.ndarray, baseline_ttft_us: int, baseline_tbt_us: int,
               policy: SloPolicy, seed: int):
    if baseline_ttft_us <= 0 or baseline_tbt_us <= 0:
        raise ValueError("baselines must be > 0")
    n = len(prompt_len)
    u1 = np.random.default_rng([seed, 10]).uniform(policy.scale_lo, policy.scale_hi, size=n)
    u2 = np.random.default_rng([seed, 11]).uniform(policy.scale_lo, policy.scale_hi, size=n)
    ttft = np.empty(n, dtype=np.int64)
    tbt = np.empty(n, dtype=np.int64)
    for k in range(n):
        f = policy.chunk_factor(int(prompt_len[k]))
        ttft[k] = max(1, int(round(baseline_ttft_us * u1[k] * f)))
        tbt[k] = max(1, int(round(baseline_tbt_us * u2[k])))
    return ttft, tbt


def assign_slos(requests: Sequence[Request], baseline_ttft_us: int, baseline_tbt_us: int,
                policy: SloPolicy, seed: int) -> None:
    prompts = np.array([r.prompt_len for r in requests], dtype=np.int64)
    ttft, tbt = slo_arrays(prompts, baseline_ttft_us, baseline_tbt_us, policy, seed)
    for r, a, b in zip(requests, ttft, tbt):
        r.slo_ttft_us = int(a)
        r.slo_tbt_us = int(b)
