"""Development aid: device step time without the L2 flush vs the per-step host API paths."""
import ctypes as C, time, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import bench
from paper_2503_13773_b200 import Engine, _native as N
import torch
reqs, cfg = bench.make_trace(0, 1)
eng = Engine(reqs, cfg, device=0)
eng.run_steps(40); eng.events
K = 20
step_ms = (C.c_double * K)(); stage_ms = (C.c_double * N.NSTAGES)()
eng._dirty(); N.check(eng._lib.co_time_steps(eng._h, K, 0, step_ms, stage_ms), "t")
print("device no-flush us/step", 1e3 * sum(step_ms) / K, {N.STAGES[q]: round(stage_ms[q] / K * 1e3, 1) for q in range(N.NSTAGES)})
eng.events; eng.step_result()
t0 = time.perf_counter()
for _ in range(K): eng.step_result()
torch.cuda.synchronize()
print("e2e us/step", (time.perf_counter() - t0) / K * 1e6)
t0 = time.perf_counter()
for _ in range(K): eng.step()
print("step() us/step", (time.perf_counter() - t0) / K * 1e6)
