"""Development aid: device engine vs the CPU oracle on many more seeded
regimes than the GPU suite holds (plain, allow_stacking, invert_amortization
and a baseline policy per seed), on one B200.

    python tools/parity_sweep.py <first_seed> <n_seeds>
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.cacheopt_oracle import CacheOptOracle  # noqa: E402
from paper_2503_13773_b200 import Engine  # noqa: E402
from tests.cases import build_product, case_params, final_arrays  # noqa: E402

POLS = ["vllm_block", "sarathi_chunked", "rlp", "s3"]


def check(p):
    reqs, cfg = build_product(p)
    eng = Engine(reqs, cfg)
    eng.run_steps(0)
    orc = CacheOptOracle(reqs, cfg)
    orc.run()
    ok = eng.events == orc.events
    fo = orc.final_state()
    ok = ok and all(np.array_equal(np.asarray(v), np.asarray(fo[k])) for k, v in final_arrays(eng).items())
    ok = ok and eng.block_tables() == orc.block_tables()
    n = len(orc.events)
    eng.close()
    return ok, n


def main():
    s0, ns = int(sys.argv[1]), int(sys.argv[2])
    t0 = time.time()
    tot = bad = events = 0
    for seed in range(s0, s0 + ns):
        base = case_params(seed)
        variants = [("plain", base),
                    ("stack", {**base, "allow_stacking": True}),
                    ("invert", {**base, "sched": {**base["sched"], "invert_amortization": True}}),
                    (POLS[seed % 4], {**base, "sched": {**base["sched"], "policy": POLS[seed % 4]}})]
        for name, p in variants:
            ok, n = check(p)
            tot += 1
            events += n
            if not ok:
                bad += 1
                print(f"MISMATCH seed {seed} {name}", flush=True)
        print(f"seed {seed}: {tot} runs, {bad} mismatches so far, {time.time() - t0:.0f} s", flush=True)
    print(f"{tot} runs ({ns} seeds x 4 variants), {events} events, {bad} mismatches, {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
