"""Request-level types of the drop-in API (the reference's core.py:26-94 and
estimation.py:18-71 shapes), materialised on the host from device arrays."""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import Enum
from typing import List, Optional

US_PER_MS = 1_000
US_PER_S = 1_000_000


def to_us(ms_value: float) -> int:
    """Milliseconds to integer microseconds, half up (core.py:21-23)."""
    return math.floor(ms_value * US_PER_MS + 0.5)


class Lifecycle(Enum):
    WAITING = "waiting"
    RUNNING = "running"
    PREEMPTED = "preempted"
    COMPLETED = "completed"


class Strategy(Enum):
    SWAP = "swap"
    RECOMPUTE = "recompute"


class Direction(Enum):
    UNDER = "under"
    OVER = "over"


# device lifecycle codes (include/cacheopt.h) -> enum; 0 = not yet arrived
STATE_FROM_CODE = {0: Lifecycle.WAITING, 1: Lifecycle.WAITING, 2: Lifecycle.RUNNING,
                   3: Lifecycle.PREEMPTED, 4: Lifecycle.COMPLETED}
STRATEGY_FROM_CODE = {0: Strategy.SWAP, 1: Strategy.RECOMPUTE}


@dataclass
class Request:
    """A serving request.  ``true_output_len`` is simulation truth that the
    planner never reads (it only sees the padded estimate)."""
    id: int
    arrival_us: int
    prompt_len: int
    true_output_len: int
    slo_ttft_us: int
    slo_tbt_us: int
    state: Lifecycle = Lifecycle.WAITING

    def __post_init__(self) -> None:
        checks = (
            (self.arrival_us >= 0, "arrival_us < 0"),
            (self.prompt_len >= 1, "prompt_len must be >= 1"),
            (self.true_output_len >= 1, "true_output_len must be >= 1"),
            (self.slo_ttft_us > 0, "slo_ttft_us must be > 0"),
            (self.slo_tbt_us > 0, "slo_tbt_us must be > 0"),
        )
        for ok, msg in checks:
            if not ok:
                raise ValueError(f"request {self.id}: {msg}")


@dataclass(frozen=True)
class LengthEstimate:
    predicted_len: int
    range_lo: int
    range_hi: int
    direction: Direction
    confidence: float
    padding: int
    estimated_len: int


@dataclass
class RequestRuntime:
    """Host snapshot of one request's device-side bookkeeping."""
    generated: int = 0
    allocated_kvc: int = 0
    used_kvc: int = 0
    first_token_at_us: Optional[int] = None
    last_token_at_us: Optional[int] = None
    max_tbt_us: int = 0
    preemption_count: int = 0
    preemption_time_us: int = 0
    estimate: Optional[LengthEstimate] = None
    kv_need: int = 0
    prefill_done: int = 0
    ready_at_us: int = 0
    preempt_started_us: int = 0
    swap_out_done_us: int = 0
    last_strategy: Optional[Strategy] = None
    first_start_us: Optional[int] = None
    completion_us: Optional[int] = None
    token_times_us: List[int] = field(default_factory=list)
