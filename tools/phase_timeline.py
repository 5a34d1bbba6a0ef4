"""Development aid: %globaltimer stamps of k_serial (planner slots 0-20,
apply slots 32-37) on config-2 window steps, as a timeline relative to the
planner's first stamp; FLUSH_L2=1 flushes L2 before every step (bench
condition).  Also prints the step's set sizes from the control block."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_13773_b200 import Engine, _native as N  # noqa: E402

reqs, cfg = bench.make_trace(0, 1, device=0)
eng = Engine(reqs, cfg)
eng.run_steps(bench.WINDOW_START)
eng.events
buf = np.zeros(64, dtype=np.int64)
N.check(eng._lib.co_phase_profile(eng._h, 1, buf.ctypes.data_as(C.POINTER(C.c_int64))), "prof")
import torch  # noqa: E402
scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for flush in (True, False):
    K = 10
    acc = np.zeros(64)
    for _ in range(K):
        if flush:
            scratch.fill_(1)
            torch.cuda.synchronize()
        buf[:] = 0
        eng.step()
        N.check(eng._lib.co_phase_profile(eng._h, 0, buf.ctypes.data_as(C.POINTER(C.c_int64))), "prof")
        acc += (buf - buf[0]).astype(np.float64)
    acc /= K * 1e3
    print(f"flush={flush}: stamp us since plan start")
    print("  " + " ".join(f"{k}:{acc[k]:.1f}" for k in range(64) if acc[k] > 0 or k == 0))
st = eng._field("STATE")
print("states", np.unique(st, return_counts=True), "live", eng._scalars().n_live)
