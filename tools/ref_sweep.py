"""Development aid (needs /root/reference): the oracle vs the UNMODIFIED
reference on the same seeds and variants tools/parity_sweep.py runs on the
device, so the device sweep is pinned to the reference transitively.

    python tools/ref_sweep.py <first_seed> <n_seeds>
"""
import copy
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")
from kvcsim.engine import Engine  # noqa: E402

from oracle.cacheopt_oracle import CacheOptOracle  # noqa: E402
from oracle.make_golden import ref_build  # noqa: E402
from tests.cases import case_params  # noqa: E402

POLS = ["vllm_block", "sarathi_chunked", "rlp", "s3"]


def main():
    s0, ns = int(sys.argv[1]), int(sys.argv[2])
    t0 = time.time()
    tot = bad = 0
    for seed in range(s0, s0 + ns):
        base = case_params(seed)
        variants = [("plain", base),
                    ("stack", {**base, "allow_stacking": True}),
                    ("invert", {**base, "sched": {**base["sched"], "invert_amortization": True}}),
                    (POLS[seed % 4], {**base, "sched": {**base["sched"], "policy": POLS[seed % 4]}})]
        for name, p in variants:
            reqs, cfg = ref_build(p)
            eng = Engine(copy.deepcopy(reqs), cfg)
            eng.run()
            orc = CacheOptOracle(reqs, cfg)
            orc.run()
            tot += 1
            if orc.events != eng.events:
                bad += 1
                print(f"MISMATCH seed {seed} {name}", flush=True)
        print(f"seed {seed}: {tot} runs, {bad} mismatches so far, {time.time() - t0:.0f} s", flush=True)
    print(f"{tot} runs ({ns} seeds x 4 variants), {bad} mismatches, {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
