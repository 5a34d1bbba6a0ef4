"""Configuration objects of the drop-in API.

Field names, defaults and validation messages follow the reference's config
dataclasses so code written against ``kvcsim`` constructs the same objects:

- ``SchedulerConfig``  scheduler.py:34-68
- ``BucketConfig``     preemption.py:19-35
- ``SwapModel`` / ``RecomputeModel``  preemption.py:81-116
- ``IterationCost`` / ``TruthCosts``  costmodel.py:17-41
- ``PredictorConfig`` / ``ConfidencePolicy``  estimation.py:23-60
- ``EngineConfig``     engine.py:65-89
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional, Tuple

US_PER_S = 1_000_000

POLICIES = ("cacheopt", "vllm_block", "rlp", "s3", "sarathi_chunked")
DEVICE_POLICIES = POLICIES
VICTIM_RULES = ("slo", "fcfs")


@dataclass(frozen=True)
class BucketConfig:
    slo_edges_us: Tuple[int, ...] = (50_000, 200_000, 500_000, 2_000_000)
    token_step: int = 128

    def __post_init__(self) -> None:
        edges = list(self.slo_edges_us)
        if edges != sorted(set(edges)):
            raise ValueError("slo_edges_us must be strictly increasing")
        if self.token_step < 1:
            raise ValueError("token_step must be >= 1")


@dataclass(frozen=True)
class SwapModel:
    """L_s(S) = gamma_s * S + delta_s [ms]."""
    gamma_s: float
    delta_s: float

    def __post_init__(self) -> None:
        if self.gamma_s <= 0:
            raise ValueError("gamma_s must be > 0")
        if self.delta_s < 0:
            raise ValueError("delta_s must be >= 0")

    def predict(self, seq_len: float) -> float:
        return self.gamma_s * seq_len + self.delta_s


@dataclass(frozen=True)
class RecomputeModel:
    """L_r(S) = alpha_r * S**beta_r + kappa_r * S + eps_r [ms]."""
    alpha_r: float
    beta_r: float
    kappa_r: float
    eps_r: float

    def __post_init__(self) -> None:
        if self.alpha_r < 0:
            raise ValueError("alpha_r must be >= 0")
        if self.beta_r <= 1:
            raise ValueError("beta_r must be > 1")
        if self.predict(1) <= 0:
            raise ValueError("model must predict positive latency for S >= 1")

    def predict(self, seq_len: float) -> float:
        return self.alpha_r * seq_len ** self.beta_r + self.kappa_r * seq_len + self.eps_r


@dataclass(frozen=True)
class IterationCost:
    base_ms: float = 5.0
    per_token_ms: float = 0.01

    def __post_init__(self) -> None:
        if self.base_ms < 0:
            raise ValueError("base_ms must be >= 0")
        if self.per_token_ms <= 0:
            raise ValueError("per_token_ms must be > 0")


@dataclass(frozen=True)
class TruthCosts:
    swap_true: SwapModel
    recompute_true: RecomputeModel

    @staticmethod
    def default() -> "TruthCosts":
        # crossover at 4000 tokens (costmodel.py:36-41)
        return TruthCosts(SwapModel(gamma_s=0.002, delta_s=8.0),
                          RecomputeModel(alpha_r=1e-6, beta_r=2.0, kappa_r=0.0, eps_r=0.0))


@dataclass
class PredictorConfig:
    bin_width: int = 50
    direction_accuracy: float = 1.0
    error_dist: str = "zero"
    error_scale: float = 0.0
    fixed_padding: Optional[int] = None
    seed: int = 0

    def __post_init__(self) -> None:
        if self.bin_width < 1:
            raise ValueError("bin_width must be >= 1")
        if not 0.0 <= self.direction_accuracy <= 1.0:
            raise ValueError("direction_accuracy must be in [0, 1]")
        if self.error_dist not in ("zero", "uniform", "normal"):
            raise ValueError(f"unknown error_dist {self.error_dist!r}")
        if self.error_scale < 0:
            raise ValueError("error_scale must be >= 0")
        if self.fixed_padding is not None and self.fixed_padding < 0:
            raise ValueError("fixed_padding must be >= 0")


@dataclass
class ConfidencePolicy:
    alpha: float = 8.0
    beta: float = 100.0
    clamp_lo: float = 0.5
    clamp_hi: float = 0.99

    def __post_init__(self) -> None:
        if self.alpha <= 0:
            raise ValueError("alpha must be > 0")
        if self.beta < 0:
            raise ValueError("beta must be >= 0")
        if not 0.0 < self.clamp_lo < self.clamp_hi < 1.0:
            raise ValueError("clamps must satisfy 0 < lo < hi < 1")


@dataclass
class SchedulerConfig:
    policy: str = "cacheopt"
    small_block_b: int = 8
    epsilon_us: int = 1_000
    token_budget: int = 2048
    preallocate_m: int = 2
    buffer_b: int = 8
    victim_rule: str = "slo"
    invert_amortization: bool = False
    decode_runway_iters: int = 6
    vllm_block_tokens: int = 32
    s3_bucket_tokens: int = 50
    rlp_padding: int = 100
    buckets: BucketConfig = field(default_factory=BucketConfig)

    def __post_init__(self) -> None:
        if self.policy not in POLICIES:
            raise ValueError(f"unknown policy {self.policy!r}, expected one of {POLICIES}")
        if self.victim_rule not in VICTIM_RULES:
            raise ValueError(f"unknown victim rule {self.victim_rule!r}")
        if self.token_budget < 1:
            raise ValueError("token_budget must be >= 1")
        if self.preallocate_m < 0:
            raise ValueError("preallocate_m must be >= 0")
        if self.decode_runway_iters < 0:
            raise ValueError("decode_runway_iters must be >= 0")
        for name in ("small_block_b", "buffer_b", "vllm_block_tokens", "s3_bucket_tokens"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        if self.rlp_padding < 0:
            raise ValueError("rlp_padding must be >= 0")
        if self.epsilon_us < 0:
            raise ValueError("epsilon_us must be >= 0")


@dataclass(frozen=True)
class KVLayout:
    """KV data plane of an instance (no reference counterpart: the reference
    only counts tokens, kvc.py:1-16).  Pages hold block_size tokens laid out
    [layer][K|V][kv_head][slot][head_dim] in bf16.  Presets: Llama-2-13B
    (40 layers, 40/40 heads) and Llama-2-70B (80 layers, 64 q / 8 kv heads)."""
    layers: int
    kv_heads: int
    q_heads: int
    head_dim: int = 128
    host_swap_pages: int = 1024
    decode: bool = True
    decode_split: int = 512

    def __post_init__(self) -> None:
        if self.layers < 1 or self.kv_heads < 1:
            raise ValueError("layers and kv_heads must be >= 1")
        if self.head_dim != 128:
            raise ValueError("head_dim must be 128")
        if self.q_heads % self.kv_heads or self.q_heads // self.kv_heads > 16:
            raise ValueError("q_heads must be a multiple (at most 16x) of kv_heads")

    @property
    def bytes_per_token(self) -> int:
        return self.layers * 2 * self.kv_heads * self.head_dim * 2

    @staticmethod
    def llama2_13b(**kw) -> "KVLayout":
        return KVLayout(layers=40, kv_heads=40, q_heads=40, **kw)

    @staticmethod
    def llama2_70b(**kw) -> "KVLayout":
        return KVLayout(layers=80, kv_heads=8, q_heads=64, **kw)


@dataclass
class EngineConfig:
    capacity_tokens: int = 16_384
    reserved_blocks: int = 8
    allow_stacking: bool = False
    sched: SchedulerConfig = field(default_factory=SchedulerConfig)
    iter_cost: IterationCost = field(default_factory=IterationCost)
    predictor: PredictorConfig = field(default_factory=PredictorConfig)
    confidence: ConfidencePolicy = field(default_factory=ConfidencePolicy)
    fixed_confidence: Optional[float] = None
    truth: TruthCosts = field(default_factory=TruthCosts.default)
    horizon_factor: int = 10
    validate_every: int = 0
    record_events: bool = True
    seed: int = 0

    def __post_init__(self) -> None:
        if self.capacity_tokens < 1:
            raise ValueError("capacity_tokens must be >= 1")
        if self.horizon_factor < 1:
            raise ValueError("horizon_factor must be >= 1")
        if self.fixed_confidence is not None and not 0.0 < self.fixed_confidence < 1.0:
            raise ValueError("fixed_confidence must be in (0, 1)")
        if self.validate_every < 0:
            raise ValueError("validate_every must be >= 0")
