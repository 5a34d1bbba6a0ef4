"""Development aid: the decode path on a small G = 8 layout with multi-tile
split-KV items (the 3-softmax-group variant), checked against fp32."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2503_13773_b200 as P  # noqa: E402
from tests.cases import build_product, case_params  # noqa: E402
from tests.kv_reference import decode_reference  # noqa: E402

lay = dict(layers=2, kv_heads=1, q_heads=8)
for seed, split in ((1, 512), (5, 300)):
    reqs, cfg = build_product(case_params(seed))
    pages = cfg.capacity_tokens // cfg.sched.small_block_b
    kv = P.KVLayout(**lay, host_swap_pages=16 * pages + 64, decode=True, decode_split=split)
    eng = P.Engine(reqs, cfg, kv=kv)
    worst, n = 0.0, 0
    for _ in range(300):
        if not eng.step():
            break
        rids, ctx, out, sid = eng.last_decode()
        for k in range(0, len(rids), max(1, len(rids) // 2)):
            ref = decode_reference(rids[k], int(ctx[k]), sid, 2, 8, 1)
            worst = max(worst, float(np.abs(out[k] - ref).max() / max(np.abs(ref).max(), 1e-6)))
            n += 1
    print(f"seed {seed} split {split}: {n} checked, worst rel err {worst:.2e}", flush=True)
