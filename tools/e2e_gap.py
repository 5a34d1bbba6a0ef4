"""Where the end-to-end step time goes: the device step with a warm L2
(co_time_steps, no flush, boundary events) vs Engine.step_result() per step
(graph launch + control-block readback + members) on the same window
(python tools/e2e_gap.py)."""
import ctypes as C
import json
import sys
import time

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_13773_b200 import Engine  # noqa: E402
from paper_2503_13773_b200 import _native as N  # noqa: E402

K = 40
reqs, cfg = bench.make_trace(0, 1, 0)
out = {}
for label in ("device_warm", "step_result", "step", "device_flush", "step_result+events"):
    eng = Engine(reqs, cfg, device=0)
    eng.run_steps(bench.WINDOW_START)
    eng.events
    if label.startswith("device"):
        step_ms = (C.c_double * K)()
        eng._dirty()
        flush = bench.L2_FLUSH_BYTES if label == "device_flush" else 0
        N.check(eng._lib.co_time_steps(eng._h, K, flush, step_ms, None), "time")
        eng._dirty()
        out[label] = round(sum(step_ms) / K * 1e3, 1)
    elif label == "step_result+events":
        eng.step_result()
        eng.events
        ts = te = 0.0
        for _ in range(K):
            t0 = time.perf_counter()
            eng.step_result()
            t1 = time.perf_counter()
            eng.events
            t2 = time.perf_counter()
            ts += t1 - t0
            te += t2 - t1
        out[label] = {"step_result_us": round(ts / K * 1e6, 1), "events_drain_us": round(te / K * 1e6, 1)}
    else:
        fn = eng.step_result if label == "step_result" else eng.step
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(K):
            fn()
        out[label] = round((time.perf_counter() - t0) / K * 1e6, 1)
    eng.close()
print(json.dumps(out))
