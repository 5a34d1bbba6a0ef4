"""Generates tests/golden/fit_golden.json from the UNMODIFIED reference's
profile -> fit -> sweet-spot pipeline (costmodel.py:73-92 sample_profile,
preemption.py:124-195 fit_swap / fit_recompute / sweet_spot), run in the
development container where /root/reference exists:

    python oracle/make_fit_golden.py

Each case is the reference's own `profile` sampling (cli.py:450-472: unique
rounded geomspace lengths, default_rng([seed, 20]), relative Gaussian noise)
of a truth model; the fixture stores the samples and the reference's fitted
coefficients and s*, which pin paper_2503_13773_b200.costprofile's restated
estimators (tests/test_costprofile.py)."""
from __future__ import annotations

import dataclasses
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REF)

from kvcsim.costmodel import TruthCosts, sample_profile  # noqa: E402
from kvcsim.preemption import RecomputeModel, SwapModel, fit_recompute, fit_swap, sweet_spot  # noqa: E402

CASES = [
    # (name, truth, min_len, max_len, points, noise, seed)
    ("default_truth", TruthCosts.default(), 16, 16384, 24, 0.05, 0),
    ("default_truth_noiseless", TruthCosts.default(), 16, 16384, 16, 0.0, 0),
    ("b200_like", TruthCosts(SwapModel(gamma_s=0.0128, delta_s=0.05),
                             RecomputeModel(alpha_r=3e-7, beta_r=2.0, kappa_r=0.017, eps_r=0.4)), 16, 8192, 12, 0.03, 7),
]


def main():
    out = []
    for name, truth, lo, hi, pts, noise, seed in CASES:
        s_values = np.unique(np.geomspace(lo, hi, pts).round().astype(int))
        rng = np.random.default_rng([seed, 20])
        rows = sample_profile(truth, [int(s) for s in s_values], noise, rng)
        swap = [(r.seq_len, r.swap_ms) for r in rows]
        rec = [(r.seq_len, r.recompute_ms) for r in rows]
        sm, rm = fit_swap(swap), fit_recompute(rec)
        try:
            spot, err = sweet_spot(rm, sm).s_star, None
        except ValueError as exc:
            spot, err = None, str(exc)
        out.append({"name": name, "swap_samples": swap, "recompute_samples": rec,
                    "swap": dataclasses.asdict(sm), "recompute": dataclasses.asdict(rm),
                    "sweet_spot": spot, "error": err})
    path = os.path.join(ROOT, "tests", "golden", "fit_golden.json")
    with open(path, "w") as fh:
        json.dump(out, fh, indent=1, sort_keys=True)
    print(f"wrote {path}: {[(c['name'], c['sweet_spot'], c['error']) for c in out]}")


if __name__ == "__main__":
    main()
