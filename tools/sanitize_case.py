"""compute-sanitizer target (tools/sanitize.sh): small regimes through every
device path -- the scheduler step graph (classify, plan, apply), the data
plane (k_data swaps/moves/fills, cooperative launch), the tcgen05 decode +
split-KV combine, device metrics and the trace generator -- with parity vs
the oracle checked at the end so a sanitizer-clean run is also a correct one.

  python tools/sanitize_case.py sched|data|stack|invert [seed] [max_steps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_13773_b200 as P  # noqa: E402
from oracle.cacheopt_oracle import CacheOptOracle  # noqa: E402
from tests.cases import build_product, case_params  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "sched"
seed = int(sys.argv[2]) if len(sys.argv) > 2 else 1
max_steps = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # 0: to the end
params = case_params(seed)
if mode == "stack":  # several guests per host; their re-homing goes through the grouped MOVE staging
    params["allow_stacking"] = True
if mode == "invert":  # invert_amortization=True: the multi-precision amortization (k_serial<., PLAN_INVERTED>)
    params["sched"] = {**params["sched"], "invert_amortization": True}
reqs, cfg = build_product(params)
kv = None
if mode in ("data", "stack"):
    pages = cfg.capacity_tokens // cfg.sched.small_block_b
    kv = P.KVLayout(layers=2, kv_heads=2, q_heads=16, host_swap_pages=16 * pages + 64, decode=True, decode_split=64)
eng = P.Engine(reqs, cfg, kv=kv)
orc = CacheOptOracle(reqs, cfg)
steps = 0
for _ in range(60):  # per-step API (the mirrored step graph)
    more = eng.step()
    orc.step()
    steps += 1
    if not more:
        break
if max_steps:
    eng.run_steps(max_steps)  # a multi-step graph
    for _ in range(max_steps):
        orc.step()
else:
    eng.run_steps(0)  # multi-step graphs to the end
    orc.run()
assert eng.events == orc.events, "device events differ from the oracle"
if kv is not None:
    bad, checked = eng.kv_verify()
    assert bad == 0, f"{bad} KV elements wrong"
if not max_steps:
    rep = eng.run()
    print(f"{mode} seed {seed}: {len(orc.events)} events identical; completed {rep.completed}")
else:
    print(f"{mode} seed {seed}: {len(orc.events)} events identical after {steps + max_steps} steps")
eng.close()
if mode == "sched":
    from paper_2503_13773_b200 import devrng
    spec = P.PRESETS["sharegpt"].sized(2000, 20.0)
    devrng.trace_arrays_device(spec, 5, 0)
    print("trace generator ok")
