"""Development aid: per-phase device time of k_plan / k_apply on config-2
window steps, from %globaltimer stamps (python tools/phase_profile.py)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_13773_b200 import Engine, _native as N  # noqa: E402
from tests.cases import config2  # noqa: E402

NAMES = ["nr/n'r", "triples", "nw embed", "demand", "victims", "grants", "decode mem", "budget", "selected",
         "proactive", "topup", "pv cache", "amortize", "claims", "extras"]

reqs, cfg = config2()
eng = Engine(reqs, cfg)
eng.run_steps(40)
buf = np.zeros(64, dtype=np.int64)
N.check(eng._lib.co_phase_profile(eng._h, 1, buf.ctypes.data_as(C.POINTER(C.c_int64))), "prof")
acc = np.zeros(64)
acc2 = np.zeros(8)
K = 10
flush = os.environ.get("FLUSH_L2") == "1"
if flush:
    import torch
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(K):
    if flush:
        scratch.fill_(1)
        torch.cuda.synchronize()
    eng.step()
    N.check(eng._lib.co_phase_profile(eng._h, 0, buf.ctypes.data_as(C.POINTER(C.c_int64))), "prof")
    acc += np.diff(np.concatenate([buf[:16], buf[32:38]]).astype(np.float64), prepend=np.nan).tolist() + [0] * 42
    acc2 += np.diff(np.array([buf[12], buf[16], buf[17], buf[18], buf[19], buf[20], buf[13]], dtype=np.float64),
                    prepend=np.nan).tolist() + [0]
d = acc[:22] / K / 1e3
for k, name in enumerate(NAMES + ["end"]):
    if k + 1 < 16:
        print(f"plan  {name:12s} {d[k + 1]:8.2f} us")
sub = acc[:0]
raw = np.array(buf)
for k, name in enumerate(["actions", "member filter", "idle/iter", "emit", "collisions+fills"]):
    print(f"apply {name:12s} {d[17 + k]:8.2f} us")

for k, name in enumerate(["ndec", "groups", "amortize(flight)", "spent", "amortize(admit)", "tail"]):
    print(f"  amortize/{name:18s} {acc2[k + 1] / K / 1e3:8.2f} us")
