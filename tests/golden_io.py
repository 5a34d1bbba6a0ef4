"""Loading tests/golden fixtures (written by oracle/make_golden.py from the
unmodified reference)."""
from __future__ import annotations

import glob
import gzip
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
TRACE_COLS = ("id", "arrival_us", "prompt_len", "true_output_len", "slo_ttft_us", "slo_tbt_us")


def names():
    """Engine-run fixtures (plan_snapshots.json.gz holds planner snapshots instead)."""
    return sorted(n for n in (os.path.basename(p)[:-8] for p in glob.glob(os.path.join(GOLDEN, "*.json.gz")))
                  if not n.startswith("plan_"))


def load(name):
    with gzip.open(os.path.join(GOLDEN, name + ".json.gz"), "rt") as fh:
        return json.load(fh)


def load_events_blob(name):
    p = os.path.join(GOLDEN, name + ".events.jsonl.gz")
    if not os.path.exists(p):
        return None
    with gzip.open(p, "rb") as fh:
        return fh.read()


def trace_digest(cols) -> str:
    h = hashlib.sha256()
    for k in TRACE_COLS:
        h.update(np.asarray(cols[k], dtype=np.int64).tobytes())
    return h.hexdigest()


def requests_from(doc):
    """Product Request objects for a fixture (stored columns, or regenerated
    with the product's trace generator when only a digest is stored)."""
    import paper_2503_13773_b200 as P
    from tests.cases import build_product
    if doc["trace"] is None:
        reqs, cfg = build_product(doc["params"])
        cols = {k: [getattr(r, k) for r in reqs] for k in TRACE_COLS}
        assert trace_digest(cols) == doc["trace_sha256"], "product trace generator diverged from the reference"
        return reqs, cfg
    t = doc["trace"]
    reqs = [P.Request(id=t["id"][k], arrival_us=t["arrival_us"][k], prompt_len=t["prompt_len"][k],
                      true_output_len=t["true_output_len"][k], slo_ttft_us=t["slo_ttft_us"][k],
                      slo_tbt_us=t["slo_tbt_us"][k]) for k in range(len(t["id"]))]
    _, cfg = build_product(doc["params"])
    return reqs, cfg


def jsonl_bytes(events) -> bytes:
    return "".join(json.dumps(e, sort_keys=True, separators=(",", ":")) + "\n" for e in events).encode()
