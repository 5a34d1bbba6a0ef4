"""Per-call device times of the trace generator at config-4 size
(python tools/tracegen_probe.py)."""
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2503_13773_b200 as P  # noqa: E402
from paper_2503_13773_b200 import devrng  # noqa: E402
from paper_2503_13773_b200.config import PredictorConfig  # noqa: E402

n = 524_288
spec = P.PRESETS["sharegpt"].sized(n, 1e6)


def t(fn, reps=5):
    fn()
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t0) * 1e3)
    return best


cols = devrng.trace_arrays_device(spec, 0)
out = {
    "raw 1M words": t(lambda: devrng.raw_device(0, 0, 1 << 20)),
    "std_exponential n": t(lambda: devrng.standard_device("exponential", 0, 0, n)),
    "std_normal n": t(lambda: devrng.standard_device("normal", 0, 1, n)),
    "trace": t(lambda: devrng.trace_arrays_device(spec, 0)),
    "slos": t(lambda: devrng.assign_slos_device(cols["prompt_len"], 2_000_000, 200_000, P.SloPolicy(), 0)),
    "pred zero": t(lambda: devrng.predictor_draws_device(PredictorConfig(), 0, n)),
    "pred uniform+flip": t(lambda: devrng.predictor_draws_device(
        PredictorConfig(error_dist="uniform", error_scale=24, direction_accuracy=0.9), 0, n)),
    "pred normal+flip": t(lambda: devrng.predictor_draws_device(
        PredictorConfig(error_dist="normal", error_scale=24, direction_accuracy=0.9), 0, n)),
}
print(json.dumps({k: round(v, 3) for k, v in out.items()}))
print(json.dumps(bench.tracegen_leg(0)))
