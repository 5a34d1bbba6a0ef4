"""CPU oracle for SURVEY.md section 8(f).3: the random streams of the trace.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2503_13773_b200`` imports or
calls this module; ``tests/`` use it as the checker of the device generator
(``csrc/trace_gen.cuh``).

The reference draws every random number of a run from numpy ``Generator``
objects (third-party dependency numpy, unpinned ``numpy>=1.24`` in the
reference's pyproject.toml:9-12; this image has numpy 2.3.5):

* ``default_rng([seed, k])`` -- SeedSequence entropy mixing, PCG64 seeding
  (workload.py:88-90, :186-187, engine.py:267);
* ``exponential(scale)`` -- the 256-layer exponential ziggurat
  (workload.py:92 inter-arrival gaps);
* ``lognormal(mu, sigma)`` = exp(mu + sigma * z), z from the 256-layer normal
  ziggurat (workload.py:96-99 prompt / output lengths);
* ``uniform(lo, hi)`` -- lo + (hi - lo) * u53 (workload.py:188-189 SLO scales);
* ``integers(-s, s + 1)`` -- Lemire's bounded draw on the 32-bit half-word
  buffer of the bit generator, ``random()`` -- u53, ``normal(0, s)``
  (estimation.py:76-99 predictor noise, one stream per run).

This module restates those published algorithms in plain Python / numpy
over the raw 64-bit PCG64 stream it generates itself, so each algorithmic
piece can be checked in isolation; ``tests/test_rng_oracle.py`` pins it
bit-for-bit against numpy's own Generator.  The ziggurat tables are the
constants numpy ships (``csrc/zig_tables.cuh``, extracted and validated by
``tools/gen_zig_tables.py``).
"""
from __future__ import annotations

import math
import os
import re
from typing import List, Sequence, Tuple

import numpy as np

M128 = (1 << 128) - 1
M64 = (1 << 64) - 1
M32 = 0xFFFFFFFF
PCG_MULT = 0x2360ED051FC65DA44385DF649FCCF645  # PCG's default 128-bit multiplier

# SeedSequence hashing constants (numpy bit_generator.pyx, after
# M.E. O'Neill's seed_seq_fe design)
INIT_A, MULT_A = 0x43B0D7E5, 0x931E8875
INIT_B, MULT_B = 0x8B51F9DD, 0x58F38DED
MIX_L, MIX_R = 0xCA01F9DD, 0x4973F715
POOL = 4


def _words(v: int) -> List[int]:
    """An entropy integer as little-endian 32-bit words (0 -> [0])."""
    if v < 0:
        raise ValueError("entropy must be non-negative")
    out = [v & M32]
    v >>= 32
    while v:
        out.append(v & M32)
        v >>= 32
    return out


def seed_sequence_state(entropy: Sequence[int], n_words64: int = 2) -> List[int]:
    """SeedSequence(entropy).generate_state(n, uint64)."""
    ent: List[int] = []
    for e in entropy:
        ent.extend(_words(int(e)))
    hc = [INIT_A]

    def hashmix(v):
        v = (v ^ hc[0]) & M32
        hc[0] = (hc[0] * MULT_A) & M32
        v = (v * hc[0]) & M32
        return v ^ (v >> 16)

    def mix(x, y):
        r = (MIX_L * x - MIX_R * y) & M32
        return r ^ (r >> 16)

    pool = [hashmix(ent[i] if i < len(ent) else 0) for i in range(POOL)]
    for s in range(POOL):
        for d in range(POOL):
            if s != d:
                pool[d] = mix(pool[d], hashmix(pool[s]))
    for s in range(POOL, len(ent)):
        for d in range(POOL):
            pool[d] = mix(pool[d], hashmix(ent[s]))
    h = INIT_B
    out32 = []
    for i in range(2 * n_words64):
        v = pool[i % POOL] ^ h
        h = (h * MULT_B) & M32
        v = (v * h) & M32
        out32.append(v ^ (v >> 16))
    return [out32[2 * i] | (out32[2 * i + 1] << 32) for i in range(n_words64)]


def pcg64_seed(entropy: Sequence[int]) -> Tuple[int, int]:
    """(state, inc) of PCG64(SeedSequence(entropy)): pcg_setseq_128_srandom_r."""
    w = seed_sequence_state(entropy, 4)
    initstate = (w[0] << 64) | w[1]
    initseq = (w[2] << 64) | w[3]
    inc = ((initseq << 1) | 1) & M128
    state = (0 * PCG_MULT + inc) & M128
    state = (state + initstate) & M128
    state = (state * PCG_MULT + inc) & M128
    return state, inc


def pcg64_raw(state: int, inc: int, n: int) -> Tuple[np.ndarray, int]:
    """n outputs (step, then XSL-RR of the new state) and the final state."""
    out = np.empty(n, dtype=np.uint64)
    for i in range(n):
        state = (state * PCG_MULT + inc) & M128
        x = ((state >> 64) ^ state) & M64
        rot = state >> 122
        out[i] = ((x >> rot) | (x << ((64 - rot) & 63))) & M64
    return out, state


def pcg64_advance(state: int, inc: int, k: int) -> int:
    """The state after k steps (LCG jump by square-and-multiply)."""
    acc_mult, acc_plus, cur_mult, cur_plus = 1, 0, PCG_MULT, inc
    while k:
        if k & 1:
            acc_mult = (acc_mult * cur_mult) & M128
            acc_plus = (acc_plus * cur_mult + cur_plus) & M128
        cur_plus = ((cur_mult + 1) * cur_plus) & M128
        cur_mult = (cur_mult * cur_mult) & M128
        k >>= 1
    return (acc_mult * state + acc_plus) & M128


def u53(w) -> float:
    """next_double: the top 53 bits scaled to [0, 1)."""
    return float(int(w) >> 11) * (1.0 / 9007199254740992.0)


# -- ziggurat tables ----------------------------------------------------------

_TABLES = None


def tables():
    """ki, wi, fi, ke, we, fe from csrc/zig_tables.cuh (hex literals)."""
    global _TABLES
    if _TABLES is None:
        here = os.path.dirname(os.path.abspath(__file__))
        src = open(os.path.join(here, "..", "paper_2503_13773_b200", "csrc", "zig_tables.cuh")).read()
        t = {}
        for name in ("ki", "wi", "fi", "ke", "we", "fe"):
            body = re.search(r"ZIG_%s\[256\]\s*=\s*\{([^}]*)\}" % name, src).group(1)
            vals = [int(x, 16) for x in re.findall(r"0x[0-9a-fA-F]+", body)]
            assert len(vals) == 256, name
            if name in ("ki", "ke"):
                t[name] = vals
            else:
                t[name] = [float(np.uint64(v).view(np.float64)) for v in vals]
        _TABLES = t
    return _TABLES


ZIG_NOR_R = 3.6541528853610088
ZIG_NOR_INV_R = 0.27366123732975828
ZIG_EXP_R = 7.69711747013104972


class Stream:
    """The bit generator's output stream with numpy's next_* semantics."""

    def __init__(self, entropy: Sequence[int], chunk: int = 4096):
        self.state, self.inc = pcg64_seed(entropy)
        self.buf = np.empty(0, dtype=np.uint64)
        self.pos = 0
        self.chunk = chunk
        self.has32 = False
        self.u32 = 0
        self.consumed = 0  # 64-bit words drawn

    def u64(self) -> int:
        if self.pos == len(self.buf):
            self.buf, self.state = pcg64_raw(self.state, self.inc, self.chunk)
            self.pos = 0
        v = int(self.buf[self.pos])
        self.pos += 1
        self.consumed += 1
        return v

    def u32_(self) -> int:
        """pcg64_next32: low half now, high half on the next call."""
        if self.has32:
            self.has32 = False
            return self.u32
        v = self.u64()
        self.has32, self.u32 = True, v >> 32
        return v & M32

    def double(self) -> float:
        return u53(self.u64())

    # distributions (numpy/random/src/distributions/distributions.c) ---------
    def std_exponential(self) -> float:
        t = tables()
        while True:
            ri = self.u64() >> 3
            idx = ri & 0xFF
            ri >>= 8
            x = ri * t["we"][idx]
            if ri < t["ke"][idx]:
                return x
            if idx == 0:
                return ZIG_EXP_R - math.log1p(-self.double())
            if (t["fe"][idx - 1] - t["fe"][idx]) * self.double() + t["fe"][idx] < math.exp(-x):
                return x

    def std_normal(self) -> float:
        t = tables()
        while True:
            r = self.u64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * t["wi"][idx]
            if sign:
                x = -x
            if rabs < t["ki"][idx]:
                return x
            if idx == 0:
                while True:
                    xx = -ZIG_NOR_INV_R * math.log1p(-self.double())
                    yy = -math.log1p(-self.double())
                    if yy + yy > xx * xx:
                        return -(ZIG_NOR_R + xx) if (rabs >> 8) & 1 else ZIG_NOR_R + xx
            elif (t["fi"][idx - 1] - t["fi"][idx]) * self.double() + t["fi"][idx] < math.exp(-0.5 * x * x):
                return x

    def bounded_int(self, low: int, high_excl: int) -> int:
        """integers(low, high) for a range below 2**32: Lemire on next_uint32."""
        rng = high_excl - 1 - low
        if rng == 0:
            return low
        if rng == M32:
            return low + self.u32_()
        excl = rng + 1
        m = self.u32_() * excl
        left = m & M32
        if left < excl:
            thr = (M32 - rng) % excl
            while left < thr:
                m = self.u32_() * excl
                left = m & M32
        return low + (m >> 32)


# -- the reference's trace / SLO / predictor draws over those streams ---------

def gen_trace(n: int, rate: float, mu_in: float, sig_in: float, lo_in: int, hi_in: int,
              mu_out: float, sig_out: float, lo_out: int, hi_out: int, seed: int):
    """workload.py:85-109 generate(): (arrival_us, prompt_len, output_len)."""
    a, p, o = Stream([seed, 0]), Stream([seed, 1]), Stream([seed, 2])
    scale = 1.0 / rate
    gaps = np.array([scale * a.std_exponential() for _ in range(n)])
    arrival = np.floor(np.cumsum(gaps) * 1_000_000 + 0.5).astype(np.int64)
    pr = np.array([math.exp(mu_in + sig_in * p.std_normal()) for _ in range(n)])
    ou = np.array([math.exp(mu_out + sig_out * o.std_normal()) for _ in range(n)])
    return (arrival, np.clip(np.rint(pr), lo_in, hi_in).astype(np.int64),
            np.clip(np.rint(ou), lo_out, hi_out).astype(np.int64))


def gen_slos(prompt_len, base_ttft: int, base_tbt: int, lo: float, hi: float, chunk_budget: int, seed: int):
    """workload.py:181-194 assign_slos()."""
    a, b = Stream([seed, 10]), Stream([seed, 11])
    rng = hi - lo
    ttft, tbt = [], []
    for pl in prompt_len:
        ut = lo + rng * a.double()
        ub = lo + rng * b.double()
        f = max(1, -(-int(pl) // chunk_budget))
        ttft.append(max(1, int(round(base_ttft * ut * f))))
        tbt.append(max(1, int(round(base_tbt * ub))))
    return np.array(ttft, dtype=np.int64), np.array(tbt, dtype=np.int64)


def gen_predictor(n: int, dist: str, scale: float, accuracy: float, seed: int):
    """estimation.py:76-99 draws, consumed per arrival in (arrival, id) order."""
    s = Stream([seed, 3])
    err = np.zeros(n, dtype=np.int32)
    flip = np.zeros(n, dtype=np.uint8)
    need_flip = accuracy < 1.0
    miss = 1.0 - accuracy
    k_int = int(scale)
    for k in range(n):
        if dist == "uniform":
            if k_int > 0:
                err[k] = s.bounded_int(-k_int, k_int + 1)
        elif dist == "normal":
            err[k] = math.floor(0.0 + scale * s.std_normal() + 0.5)
        if need_flip:
            flip[k] = 1 if s.double() < miss else 0
    return err, flip
