"""Development aid: the config-2 window (bench workload) on one B200.

  python tools/step_probe.py time    # step / stage times, L2 flushed and warm
  python tools/step_probe.py ncu     # 3 flushed window steps (for ncu -k ... -s 40)
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_13773_b200 import Engine, _native as N  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "time"
reqs, cfg = bench.make_trace(0, 1, device=0)
K = int(os.environ.get("K", "20"))


def window(stages: bool, flush: int):
    eng = Engine(reqs, cfg)
    eng.run_steps(bench.WINDOW_START)
    eng.events
    step = (C.c_double * K)()
    st = (C.c_double * N.NSTAGES)()
    eng._dirty()
    N.check(eng._lib.co_time_steps(eng._h, K, flush, step, st if stages else None), "co_time_steps")
    eng.close()
    return sum(step) / K * 1e3, {N.STAGES[q]: round(st[q] / K * 1e3, 2) for q in range(N.NSTAGES)}


if mode == "time":
    for flush in (bench.L2_FLUSH_BYTES, 0):
        t, _ = window(False, flush)
        t2, s = window(True, flush)
        print(f"flush={flush >> 20}MiB step {t:.1f} us | staged {t2:.1f} us {s}")
else:
    eng = Engine(reqs, cfg)
    eng.run_steps(bench.WINDOW_START)
    step = (C.c_double * 3)()
    eng._dirty()
    flush = int(os.environ.get("FLUSH", bench.L2_FLUSH_BYTES))  # FLUSH=0: warm-L2 steps
    N.check(eng._lib.co_time_steps(eng._h, 3, flush, step, None), "co_time_steps")
    print("steps us", [round(x * 1e3, 1) for x in step])
