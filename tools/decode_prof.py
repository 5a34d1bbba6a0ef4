"""Development aid: per-role wait cycles of k_decode_tc05 (CTA 0) from a
-DT5_PROF build (CACHEOPT_LIB=...), config-5 decode steps."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2503_13773_b200 as P  # noqa: E402
from paper_2503_13773_b200 import _native as N  # noqa: E402

kv = P.KVLayout.llama2_70b(host_swap_pages=4096, decode=True, decode_split=512)
cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16),
                     record_events=False)
eng = P.Engine(bench.long_output_trace(), cfg, device=0, kv=kv)
eng.set_decode(False)
eng.run_steps(3000)
eng.set_decode(True)
buf = np.zeros(64, dtype=np.int64)
N.check(eng._lib.co_phase_profile(eng._h, 1, buf.ctypes.data_as(C.POINTER(C.c_int64))), "prof")
for _ in range(5):
    eng.step()
N.check(eng._lib.co_phase_profile(eng._h, 0, buf.ctypes.data_as(C.POINTER(C.c_int64))), "prof")
names = ["sm: wait S", "sm: ld+max", "sm: named bar", "sm: P write+arrive", "sm: wait O", "sm: fold total",
         "mma: wait K", "mma: wait S-empty", "mma: wait P", "mma: wait O-empty+V", "sm: tiles", "prod K: wait slot",
         "prod V: wait slot", "mma: S latency", "mma: O latency"]
tiles = max(buf[58], 1)
for k, n in enumerate(names):
    print(f"{n:22s} {buf[48 + k]:>14d}  per sm-tile {buf[48 + k] / tiles:10.1f}")
