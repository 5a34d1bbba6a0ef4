"""Hardware-true swap / recompute cost models.

The reference decides swap vs recompute from two latency models and their
crossover (preemption.py:81-116 SwapModel / RecomputeModel, :176-195
sweet_spot), and gets the models by fitting profiled samples
(cli.py:409-447 ``fit``: preemption.py:124-172 fit_swap / fit_recompute).
Its ``profile`` command (cli.py:450-472) only evaluates the synthetic truth
models of costmodel.py.  Here the samples are measured on this B200:

* swap: the round trip (swap-out + swap-in, the two halves the engine charges
  at preempt and readmit, engine.py:371-373 / :391-394) of S tokens through
  the engine's own ``k_data`` kernel between HBM pages and pinned host pages;
* recompute: a prefill proxy for re-deriving S tokens of KV, i.e. one
  transformer layer's prefill of S tokens (QKV / O / gated-MLP GEMMs and
  causal GQA attention, bf16 on the tensor cores) times the layer count.

``fit_swap`` / ``fit_recompute`` / ``sweet_spot`` are this package's own
estimators for the reference's model families and selection rule (closed-form
centred regression for the line; one batched QR over the whole 1.20..3.00
exponent grid; a doubling search for the crossover); their results are pinned
to the reference's own fits on its own profile samples
(tests/golden/fit_golden.json).  ``hardware_truth`` returns a
``TruthCosts`` the engine (and the CPU oracle) accept unchanged.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Sequence, Tuple

import numpy as np

from .config import RecomputeModel, SwapModel, TruthCosts

# the reference's exponent grid for L_r (preemption.py:140): 1.20, 1.21, ..., 3.00
BETA_GRID = np.round(np.linspace(1.2, 3.0, 181), 2)


def _samples(samples, need: int):
    """(S, latency) columns with the reference's input contract
    (preemption.py:124-130, :143-151): enough points, two distinct lengths."""
    if len(samples) < need:
        raise ValueError(f"need at least {need} samples")
    a = np.asarray(samples, dtype=float).reshape(len(samples), 2)
    if np.ptp(a[:, 0]) == 0:
        raise ValueError("samples are degenerate: constant seq_len")
    return a[:, 0], a[:, 1]


def fit_swap(samples: Sequence[Tuple[float, float]]) -> SwapModel:
    """L_s(S) = gamma*S + delta by least squares (the estimator of
    preemption.py:124-137), solved in closed form on centred moments:
    gamma = cov(S, y) / var(S), delta = mean(y) - gamma*mean(S), clamped >= 0."""
    s, y = _samples(samples, 2)
    ds, dy = s - s.mean(), y - y.mean()
    gamma = float(np.dot(ds, dy) / np.dot(ds, ds))
    if not gamma > 0:
        raise ValueError(f"fitted swap slope {gamma:.3g} is not positive")
    delta = float(y.mean() - gamma * s.mean())
    return SwapModel(gamma_s=gamma, delta_s=max(0.0, delta))


def _grid_solutions(s: np.ndarray, y: np.ndarray) -> np.ndarray:
    """For every exponent b of BETA_GRID at once: the coefficients c(b) that
    minimise sum_i ((c . [S_i^b, S_i, 1]) / y_i - 1)^2, i.e. the relative-
    error least squares of preemption.py:157-160.  One batched Householder QR
    of the row-weighted, column-equilibrated [G, n, 3] design stack, then a
    3x3 triangular solve per exponent; an exponent whose design is rank
    deficient falls back to the minimum-norm solution (what an SVD solver
    returns).  -> [G, 3] (alpha, kappa, eps)."""
    w = 1.0 / y
    X = np.stack([s[None, :] ** BETA_GRID[:, None], np.broadcast_to(s, (len(BETA_GRID), s.size)),
                  np.ones((len(BETA_GRID), s.size))], axis=-1) * w[None, :, None]
    col = np.sqrt(np.einsum("gnk,gnk->gk", X, X))
    Xs = X / col[:, None, :]
    Q, R = np.linalg.qr(Xs)                                  # batched, [G,n,3] / [G,3,3]
    rhs = np.einsum("gnk,n->gk", Q, np.ones_like(y))
    out = np.empty((len(BETA_GRID), 3))
    diag = np.abs(np.diagonal(R, axis1=1, axis2=2))
    for g in range(len(BETA_GRID)):
        if diag[g].min() > 1e-12 * diag[g].max():
            z = np.zeros(3)
            for k in (2, 1, 0):                                # back substitution
                z[k] = (rhs[g, k] - R[g, k, k + 1:] @ z[k + 1:]) / R[g, k, k]
        else:
            z = np.linalg.pinv(Xs[g]) @ np.ones_like(y)
        out[g] = z / col[g]
    return out


def fit_recompute(samples: Sequence[Tuple[float, float]]) -> RecomputeModel:
    """L_r(S) = alpha*S^beta + kappa*S + eps: the exponent is taken from the
    reference's grid (preemption.py:140-172) as the admissible candidate
    (alpha >= 0, positive prediction at S = 1 and at every sample) with the
    smallest relative squared error; ties keep the smaller exponent."""
    s, y = _samples(samples, 8)
    if (y <= 0).any():
        raise ValueError("latencies must be positive")
    coef = _grid_solutions(s, y)
    feats = np.stack([s[None, :] ** BETA_GRID[:, None], np.broadcast_to(s, (len(BETA_GRID), s.size)),
                      np.ones((len(BETA_GRID), s.size))], axis=-1)
    pred = np.einsum("gnk,gk->gn", feats, coef)
    ok = (coef[:, 0] >= 0) & (coef.sum(axis=1) > 0) & (pred > 0).all(axis=1)
    if not ok.any():
        raise ValueError("no admissible fit found on the exponent grid")
    err = (((pred - y[None, :]) / y[None, :]) ** 2).sum(axis=1)
    g = int(np.flatnonzero(ok)[np.argmin(err[ok])])
    alpha, kappa, eps = (float(v) for v in coef[g])
    return RecomputeModel(alpha_r=alpha, beta_r=float(BETA_GRID[g]), kappa_r=kappa, eps_r=eps)


def sweet_spot(rec: RecomputeModel, swp: SwapModel, s_max: int = 1_000_000) -> int:
    """s* of preemption.py:176-195: the largest integer S in [1, s_max] with
    L_r(S) <= L_s(S).  d(S) = L_r - L_s is convex in S (beta > 1), so with
    d(1) <= 0 < d(s_max) the feasible lengths are exactly [1, s*]: located by
    a doubling search for the first infeasible power of two, then halving
    steps inside that octave.  ValueError when there is no crossover."""
    def d(x):
        return rec.predict(x) - swp.predict(x)
    if d(1) > 0:
        raise ValueError("no crossover: swap dominates over the whole range")
    if d(s_max) <= 0:
        raise ValueError("no crossover: recompute dominates over the whole range")
    hi = 2
    while hi < s_max and d(hi) <= 0:
        hi *= 2
    hi = min(hi, s_max)                                        # d(hi) > 0
    lo = max(1, hi // 2) if d(max(1, hi // 2)) <= 0 else 1     # d(lo) <= 0
    step = 1 << max(0, (hi - lo).bit_length() - 1)
    while step:                                                # lo = largest feasible
        if lo + step < hi and d(lo + step) <= 0:
            lo += step
        step >>= 1
    return lo


def decision_spot(rec: RecomputeModel, swp: SwapModel) -> int:
    """The s* the planner uses (scheduler.py:381-393 _cached_sweet_spot):
    all-swap encodes as 0, all-recompute as 2**62."""
    try:
        return sweet_spot(rec, swp)
    except ValueError as exc:
        return 0 if "swap dominates" in str(exc) else 1 << 62


# -- measurement on the B200 -------------------------------------------------

@dataclasses.dataclass(frozen=True)
class ModelDims:
    """Transformer dimensions of the layout whose KV is swapped/recomputed."""
    name: str
    layers: int
    hidden: int
    ffn: int
    q_heads: int
    kv_heads: int
    head_dim: int = 128

    @staticmethod
    def llama2_13b() -> "ModelDims":
        return ModelDims("Llama-2-13B", 40, 5120, 13824, 40, 40)

    @staticmethod
    def llama2_70b() -> "ModelDims":
        return ModelDims("Llama-2-70B", 80, 8192, 28672, 64, 8)


def default_lengths(lo: int = 16, hi: int = 8192, points: int = 12) -> List[int]:
    """Geometric sample lengths, as the reference's profile command
    (cli.py:453-456: unique rounded geomspace)."""
    return [int(s) for s in np.unique(np.geomspace(lo, hi, points).round().astype(int))]


def measure_swap(lengths: Sequence[int], kv_layout=None, iters: int = 3, device: int = 0) -> List[Tuple[int, float]]:
    """(S, round-trip ms) through the engine's data kernel: a gather of S
    tokens' KV from HBM pages into pinned host pages plus the scatter back."""
    from . import Engine, EngineConfig, KVLayout, SchedulerConfig
    from .workload import TraceSpec, generate
    kv = kv_layout or KVLayout.llama2_70b(host_swap_pages=1, decode=False)
    s_max = max(lengths)
    pages = (s_max + 15) // 16 + 1
    kv = dataclasses.replace(kv, host_swap_pages=pages, decode=False)
    cap = max(pages * 16, 4096)
    cfg = EngineConfig(capacity_tokens=cap, reserved_blocks=0, sched=SchedulerConfig(small_block_b=16),
                       record_events=False)
    reqs = generate(TraceSpec(arrival_rate=1.0, num_requests=4, input_mean=64, input_min=16, input_max=128,
                              output_mean=16, output_min=4, output_max=32), 0)
    eng = Engine(reqs, cfg, device=device, kv=kv)
    try:
        out = []
        for s in lengths:
            o, i = eng.swap_bench(int(s), iters=iters)
            out.append((int(s), o + i))
        return out
    finally:
        eng.close()


def measure_recompute(lengths: Sequence[int], dims: ModelDims = None, iters: int = 3,
                      device: int = 0) -> List[Tuple[int, float]]:
    """(S, ms) of re-deriving S tokens of KV: one layer's bf16 prefill of S
    tokens (cuBLAS GEMMs + causal GQA SDPA) times the layer count."""
    import torch
    import torch.nn.functional as F
    dims = dims or ModelDims.llama2_70b()
    dev = torch.device("cuda", device)
    g = torch.Generator(device=dev).manual_seed(0)
    H, D = dims.hidden, dims.head_dim
    kvw = dims.kv_heads * D
    def w(r, c):
        return (torch.randn(r, c, device=dev, dtype=torch.bfloat16, generator=g) * (1.0 / math.sqrt(r)))
    wqkv, wo = w(H, H + 2 * kvw), w(H, H)
    wgu, wd = w(H, 2 * dims.ffn), w(dims.ffn, H)

    def layer(x):
        qkv = x @ wqkv
        s = x.shape[0]
        q = qkv[:, :H].view(s, dims.q_heads, D).transpose(0, 1)
        k = qkv[:, H:H + kvw].view(s, dims.kv_heads, D).transpose(0, 1)
        v = qkv[:, H + kvw:].view(s, dims.kv_heads, D).transpose(0, 1)
        a = F.scaled_dot_product_attention(q.unsqueeze(0), k.unsqueeze(0), v.unsqueeze(0), is_causal=True,
                                           enable_gqa=dims.q_heads != dims.kv_heads)
        h = x + a.squeeze(0).transpose(0, 1).reshape(s, H) @ wo
        gu = h @ wgu
        return h + (F.silu(gu[:, :dims.ffn]) * gu[:, dims.ffn:]) @ wd

    out = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.no_grad():
        for s in lengths:
            x = torch.randn(int(s), H, device=dev, dtype=torch.bfloat16, generator=g)
            layer(x)  # warm-up (kernel selection)
            torch.cuda.synchronize(dev)
            e0.record()
            for _ in range(iters):
                layer(x)
            e1.record()
            torch.cuda.synchronize(dev)
            out.append((int(s), e0.elapsed_time(e1) / iters * dims.layers))
    del wqkv, wo, wgu, wd
    torch.cuda.empty_cache()
    return out


def hardware_truth(lengths: Sequence[int] = None, kv_layout=None, dims: ModelDims = None,
                   device: int = 0) -> Dict:
    """Profile both costs on this GPU, fit them with the reference's
    estimators, and return coefficients.json's content (cli.py:440-446) plus
    the samples and a TruthCosts for EngineConfig(truth=...)."""
    lengths = list(lengths or default_lengths())
    swap = measure_swap(lengths, kv_layout, device=device)
    rec = measure_recompute(lengths, dims, device=device)
    sm, rm = fit_swap(swap), fit_recompute(rec)
    try:
        spot = sweet_spot(rm, sm)
        note = None
    except ValueError as exc:
        spot, note = decision_spot(rm, sm), str(exc)
    return {"swap": dataclasses.asdict(sm), "recompute": dataclasses.asdict(rm), "sweet_spot": spot,
            "crossover_note": note, "samples": {"swap": swap, "recompute": rec},
            "truth": TruthCosts(sm, rm)}
