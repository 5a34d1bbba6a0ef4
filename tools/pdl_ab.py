"""A/B of programmatic dependent launch in the step graph (config-2 window,
L2 flushed per step): step time with boundary-only events, PDL on / off, and
with stage events (python tools/pdl_ab.py)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_13773_b200 import Engine  # noqa: E402
from paper_2503_13773_b200 import _native as N  # noqa: E402

K = 20
out = {}
reqs, cfg = bench.make_trace(0, 1, 0)
for label, pdl, stages in (("pdl", "1", False), ("no_pdl", "0", False), ("pdl_stage_events", "1", True),
                           ("pdl2", "1", False), ("no_pdl2", "0", False)):
    os.environ["CACHEOPT_PDL"] = pdl
    eng = Engine(reqs, cfg, device=0)
    eng.run_steps(bench.WINDOW_START)
    eng.events
    step_ms = (C.c_double * K)()
    stage_ms = (C.c_double * N.NSTAGES)()
    torch.cuda.synchronize()
    eng._dirty()
    N.check(eng._lib.co_time_steps(eng._h, K, bench.L2_FLUSH_BYTES, step_ms, stage_ms if stages else None),
            "time")
    eng._dirty()
    out[label] = round(sum(step_ms) / K * 1e3, 2)
    eng.close()
print(json.dumps(out))
