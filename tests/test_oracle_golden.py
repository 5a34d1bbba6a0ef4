"""The CPU oracle against golden vectors produced by the unmodified reference
(oracle/make_golden.py): byte-identical event logs, per-request outcomes,
pool totals and utilisation samples."""
import hashlib
import json

import numpy as np
import pytest

from oracle.cacheopt_oracle import CacheOptOracle
from tests import golden_io as G

CASES = G.names()


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_reference_fixture(name):
    doc = G.load(name)
    reqs, cfg = G.requests_from(doc)
    orc = CacheOptOracle(reqs, cfg)
    if doc["steps"] is None:
        orc.run()
    else:
        for _ in range(doc["steps"]):
            orc.step()
    blob = G.jsonl_bytes(orc.events)
    ref_blob = G.load_events_blob(name)
    if ref_blob is not None and blob != ref_blob:
        a, b = blob.decode().splitlines(), ref_blob.decode().splitlines()
        k = next(i for i, (x, y) in enumerate(zip(a, b)) if x != y)
        raise AssertionError(f"first differing event {k}:\n oracle {a[k]}\n ref    {b[k]}")
    assert hashlib.sha256(blob).hexdigest() == doc["events_sha256"]
    fo = orc.final_state()
    names = {"generated": "generated", "preemption_count": "preemption_count",
             "preemption_time_us": "preemption_time_us", "max_tbt_us": "max_tbt_us", "kv_need": "kv_need",
             "prefill_done": "prefill_done", "used": "used", "completion_us": "completion_us",
             "first_token_at_us": "first_token_at_us"}
    for ref_key, orc_key in names.items():
        assert np.array_equal(fo[orc_key], np.asarray(doc["final"][ref_key])), ref_key
    assert (orc.fp_sum, orc.used_sum, orc.rsv_cur) == (
        doc["pool"]["footprint"], doc["pool"]["used"], doc["pool"]["reserved"])
    samples = [list(s) for s in orc.samples]
    assert hashlib.sha256(json.dumps(samples).encode()).hexdigest() == doc["samples_sha256"]
    if doc.get("metrics") is not None:
        # engine.py:132-211 + :662-671: the reference's own MetricsReport, exact
        assert orc.metrics() == doc["metrics"]


def test_metrics_fixtures_present():
    """Every full-run fixture carries the reference's MetricsReport."""
    full = [n for n in CASES if G.load(n)["steps"] is None]
    assert len(full) >= 18
    for n in full:
        assert G.load(n).get("metrics"), n


def test_fixture_set_covers_the_decision_kinds():
    kinds = set()
    for name in CASES:
        blob = G.load_events_blob(name)
        if blob is None:
            continue
        for line in blob.decode().splitlines():
            e = json.loads(line)
            kinds.add(e["ev"] if e["ev"] != "preempt" else f"preempt/{e['cause']}/{e['strategy']}")
    for k in ("arrive", "admit", "iter", "complete", "readmit", "preempt/plan/recompute", "preempt/plan/swap"):
        assert k in kinds, k


@pytest.mark.parametrize("name", [n for n in CASES if n.startswith("case")][:5])
def test_block_tables_conserve_pages_every_step(name):
    """N1 restatement invariants (no reference counterpart): every standalone
    record owns exactly fp(granted)/bs distinct pages, every page is owned
    once or free, checked after every step of a golden scenario."""
    doc = G.load(name)
    reqs, cfg = G.requests_from(doc)
    orc = CacheOptOracle(reqs, cfg)
    while orc.step():
        orc.check_invariants()
    orc.check_invariants()
    tabs, free = orc.block_tables()
    standalone = {orc.rid[i] for i in range(orc.n) if orc.holds[i] and orc.host[i] < 0 and orc.granted[i] > 0}
    assert set(tabs) == standalone
    assert sorted(free + [p for t in tabs.values() for p in t]) == list(range(orc.n_pages))
