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

``fit_swap`` / ``fit_recompute`` / ``sweet_spot`` restate the reference's
fitting code (numpy least squares, the same 1.20..3.00 exponent grid) so the
fitted models -- and hence every decision and charge -- match what the
reference would derive from the same samples.  ``hardware_truth`` returns a
``TruthCosts`` the engine (and the CPU oracle) accept unchanged.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Sequence, Tuple

import numpy as np

from .config import RecomputeModel, SwapModel, TruthCosts

# preemption.py:140: exponent grid of fit_recompute
BETA_GRID = [round(1.2 + 0.01 * k, 2) for k in range(181)]


def fit_swap(samples: Sequence[Tuple[float, float]]) -> SwapModel:
    """OLS line latency_ms = gamma * S + delta (preemption.py:124-137)."""
    if len(samples) < 2:
        raise ValueError("need at least 2 samples")
    s = np.asarray([p[0] for p in samples], dtype=float)
    y = np.asarray([p[1] for p in samples], dtype=float)
    if np.unique(s).size < 2:
        raise ValueError("samples are degenerate: constant seq_len")
    design = np.column_stack([s, np.ones_like(s)])
    (gamma, delta), *_ = np.linalg.lstsq(design, y, rcond=None)
    if gamma <= 0:
        raise ValueError(f"fitted swap slope {gamma:.3g} is not positive")
    return SwapModel(gamma_s=float(gamma), delta_s=float(max(0.0, delta)))


def fit_recompute(samples: Sequence[Tuple[float, float]]) -> RecomputeModel:
    """Exponent grid search, relative-error-weighted least squares per
    candidate, minimum residual (preemption.py:143-172)."""
    if len(samples) < 8:
        raise ValueError("need at least 8 samples")
    s = np.asarray([p[0] for p in samples], dtype=float)
    y = np.asarray([p[1] for p in samples], dtype=float)
    if np.unique(s).size < 2:
        raise ValueError("samples are degenerate: constant seq_len")
    if np.any(y <= 0):
        raise ValueError("latencies must be positive")
    w = 1.0 / y
    best, best_resid = None, np.inf
    for beta in BETA_GRID:
        design = np.column_stack([s ** beta, s, np.ones_like(s)])
        coeffs, *_ = np.linalg.lstsq(design * w[:, None], np.ones_like(y), rcond=None)
        alpha, kappa, eps = (float(c) for c in coeffs)
        if alpha < 0 or alpha + kappa + eps <= 0:
            continue
        pred = design @ np.array([alpha, kappa, eps])
        if np.any(pred <= 0):
            continue
        resid = float(np.sum(((pred - y) * w) ** 2))
        if resid < best_resid:
            best_resid, best = resid, (alpha, beta, kappa, eps)
    if best is None:
        raise ValueError("no admissible fit found on the exponent grid")
    alpha, beta, kappa, eps = best
    return RecomputeModel(alpha_r=alpha, beta_r=beta, kappa_r=kappa, eps_r=eps)


def sweet_spot(rec: RecomputeModel, swp: SwapModel, s_max: int = 1_000_000) -> int:
    """Largest S with recompute no slower than swap, bisection to +-1 token
    (preemption.py:176-195); ValueError without a crossover, as there."""
    def diff(s):
        return rec.predict(s) - swp.predict(s)
    lo, hi = 1, s_max
    if diff(lo) > 0:
        raise ValueError("no crossover: swap dominates over the whole range")
    if diff(hi) <= 0:
        raise ValueError("no crossover: recompute dominates over the whole range")
    while hi - lo > 1:
        mid = (lo + hi) // 2
        lo, hi = (mid, hi) if diff(mid) <= 0 else (lo, mid)
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
