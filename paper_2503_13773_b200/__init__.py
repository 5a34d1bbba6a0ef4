"""B200-native CacheOPT hot path (arXiv 2503.13773) behind the reference
simulator's Engine API.  The compute path is libcacheopt.so (sm_100a CUDA,
include/cacheopt.h); this package is the host-side mirror of the reference's
interface: config objects, trace input, and the Engine drop-in."""
from .config import (BucketConfig, ConfidencePolicy, EngineConfig, IterationCost, KVLayout, PredictorConfig,
                     RecomputeModel, SchedulerConfig, SwapModel, TruthCosts)
from .core import Direction, LengthEstimate, Lifecycle, Request, RequestRuntime, Strategy, to_us
from .engine import (Engine, MetricsReport, PoolView, calibrate_slo_baselines, compute_metrics,
                     write_events_jsonl)
from .workload import PRESETS, SloPolicy, TraceSpec, assign_slos, generate, ingest_csv, trace_arrays

__version__ = "0.1.0"
