"""Development aid / bench evidence: BASELINE config 3 (2x-rate heavy
preemption) with the B200-fitted Llama-2-70B swap/recompute models (swap at
every length) and the 70B KV data plane WITH the paged decode on, run to the
end in windows of K timed steps (stage events), split swap I/O on vs off:
step time, data / decode stage times, swapped bytes and in-run swap GB/s.

  python tools/swap_probe.py [K]"""
import ctypes as C
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_13773_b200 as P  # noqa: E402
from paper_2503_13773_b200 import _native as N  # noqa: E402
from tests.cases import config3  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 500
# the 70B fit of profiles/r01/costmodel (bench costmodel leg): swap dominates, s* = 0
truth = P.TruthCosts(P.SwapModel(0.01287, 0.0), P.RecomputeModel(0.0131, 1.2, 0.0285, 23.55))
res = {}
for split in ("1", "0"):
    os.environ["CACHEOPT_SPLIT_IO"] = split
    reqs, cfg = config3()
    cfg = dataclasses.replace(cfg, truth=truth, record_events=False)
    kv = P.KVLayout.llama2_70b(host_swap_pages=2048, decode=True, decode_split=512)
    eng = P.Engine(reqs, cfg, device=0, kv=kv)
    step_ms = (C.c_double * K)()
    stage_ms = (C.c_double * N.NSTAGES)()
    tot_step, tot_stage, windows = 0.0, [0.0] * N.NSTAGES, 0
    while not eng._scalars().done:
        eng._dirty()
        N.check(eng._lib.co_time_steps(eng._h, K, 0, step_ms, stage_ms), "co_time_steps")
        tot_step += sum(step_ms)
        tot_stage = [a + b for a, b in zip(tot_stage, stage_ms)]
        windows += 1
        eng._dirty()
    st = eng.data_stats()
    io = eng.swap_io_stats()
    bad, checked = eng.kv_verify()
    stages = dict(zip(N.STAGES, tot_stage))
    res[split] = {"split_io": split == "1", "steps": eng._scalars().steps, "step_ms_total": tot_step,
                  "data_stage_ms": stages["data"], "decode_stage_ms": stages["decode"],
                  "swap_out_gb": st["swap_out_bytes"] / 1e9, "swap_in_gb": st["swap_in_bytes"] / 1e9,
                  "decode_member_steps": st["decode_member_steps"], "io": io,
                  "kv_integrity": {"mismatches": bad, "checked": checked}}
    print(json.dumps(res[split]), flush=True)
    eng.close()
