"""BASELINE config 5 end to end on the device: the long-output trace with the
Llama-2-70B KV data plane and the paged decode ON for every step, the
default truth costs (s* = 4000: long sequences swap), run to completion in
windows of K timed steps (stage events); split swap I/O on vs off.  Reports
step / data / decode stage times, swapped bytes, in-run swap GB/s (k_swapio
device time) and KV integrity.

  python tools/config5_run.py [K]"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2503_13773_b200 as P  # noqa: E402
from paper_2503_13773_b200 import _native as N  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
for split in ("1", "0"):
    os.environ["CACHEOPT_SPLIT_IO"] = split
    kv = P.KVLayout.llama2_70b(host_swap_pages=16384, decode=True, decode_split=512)
    cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16),
                         record_events=False)
    eng = P.Engine(bench.long_output_trace(), cfg, device=0, kv=kv)
    step_ms = (C.c_double * K)()
    stage_ms = (C.c_double * N.NSTAGES)()
    tot, stages, bad, checked = 0.0, [0.0] * N.NSTAGES, 0, 0
    while not eng._scalars().done:
        eng._dirty()
        N.check(eng._lib.co_time_steps(eng._h, K, 0, step_ms, stage_ms), "co_time_steps")
        tot += sum(step_ms)
        stages = [a + b for a, b in zip(stages, stage_ms)]
        eng._dirty()
        b, c = eng.kv_verify()
        bad, checked = bad + b, checked + c
    st = eng.data_stats()
    io = eng.swap_io_stats()
    rep = eng.run()
    sd = dict(zip(N.STAGES, stages))
    out = {"split_io": split == "1", "steps": eng._scalars().steps, "step_ms_total": tot,
           "data_stage_ms": sd["data"], "decode_stage_ms": sd["decode"],
           "preemptions": rep.preemption_total, "completed": rep.completed,
           "swap_out_gb": st["swap_out_bytes"] / 1e9, "swap_in_gb": st["swap_in_bytes"] / 1e9,
           "decode_member_steps": st["decode_member_steps"], "decode_ctx_tokens": st["decode_ctx_tokens"],
           "io": io, "kv_integrity": {"mismatches": bad, "checked": checked}}
    print(json.dumps(out), flush=True)
    eng.close()
