"""plan_batch(PlannerInputs, cfg) (scheduler.py:939-950) on the device against
BatchPlans the UNMODIFIED reference returned on the same snapshots
(tests/golden/plan_snapshots.json.gz, oracle/make_plan_golden.py): 120
snapshots from 15 runs -- cacheopt with preemptions, embeddings, reserve
draws, claims and deferrals, stacking, invert_amortization, and the four
baseline policies."""
import gzip
import json
import os

import pytest

from paper_2503_13773_b200 import BucketConfig, IterationCost, Lifecycle, RecomputeModel, SchedulerConfig, SwapModel

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "plan_snapshots.json.gz")


def _snaps():
    with gzip.open(GOLDEN, "rt") as fh:
        return json.load(fh)


class SnapshotPool:
    """The read-only BlockPool queries plan_batch makes (kvc.py:88-152)."""

    def __init__(self, doc):
        self.capacity, self.block_size = doc["capacity"], doc["block_size"]
        self.reserved_target, self.buffer_b = doc["reserved_target"], doc["buffer_b"]
        self.allow_stacking = doc["allow_stacking"]
        self.reserved_blocks_current = doc["reserved_current"]
        self._r = {r["id"]: r for r in doc["records"]}
        self._order = [r["id"] for r in doc["records"]]

    def owners(self):
        return list(self._order)

    def granted_of(self, i):
        return self._r[i]["granted"]

    def host_of(self, i):
        return self._r[i]["host"]

    def offset_of(self, i):
        return self._r[i]["offset"]

    def guests_of(self, i):
        return list(self._r[i]["guests"])

    def reserved_drawn_of(self, i):
        return self._r[i]["reserved"]

    def used_of(self, i):
        return self._r[i]["used"]


def test_fixture_covers_the_plan_kinds():
    snaps = _snaps()
    assert len(snaps) >= 90
    acts = {a[0] for s in snaps for a in s["plan"]["actions"]}
    assert {"allocate", "grow", "embed", "reserve"} <= acts
    assert any(s["plan"]["preempt"] for s in snaps) and any(s["plan"]["claims"] for s in snaps)
    assert any(s["plan"]["deferred"] for s in snaps)
    assert {s["sched"]["policy"] for s in snaps} == {"cacheopt", "vllm_block", "sarathi_chunked", "rlp", "s3"}
    assert sum(1 for s in snaps if s["sched"]["invert_amortization"]) >= 24


@pytest.mark.gpu
@pytest.mark.parametrize("k", list(range(120)))
def test_device_plan_batch_equals_reference_plan(cuda_ok, k):
    from paper_2503_13773_b200.scheduler import PlannerInputs, ReqView, plan_batch
    s = _snaps()[k]

    def view(d):
        d = dict(d)
        d["state"] = Lifecycle(d["state"])
        return ReqView(**d)

    sched = dict(s["sched"])
    cfg = SchedulerConfig(**sched, buckets=BucketConfig(tuple(s["buckets"]["slo_edges_us"]), s["buckets"]["token_step"]))
    inp = PlannerInputs(waiting=[view(v) for v in s["waiting"]], running=[view(v) for v in s["running"]],
                        pool=SnapshotPool(s["pool"]), t_i_max_us=s["t_i_max_us"], iter_cost=IterationCost(**s["iter_cost"]),
                        swap_model=SwapModel(**s["swap_model"]), recompute_model=RecomputeModel(**s["recompute_model"]))
    plan = plan_batch(inp, cfg)
    want = s["plan"]
    assert [[m.req_id, m.tokens] for m in plan.members] == want["members"], s["run"]
    assert plan.batch_tokens == want["batch_tokens"]
    assert [[i, st.value] for i, st in plan.preempt] == want["preempt"]
    got_acts = [[a.kind, a.req_id, a.tokens, a.blocks,
                 None if a.quote is None else [a.quote.host, a.quote.start_offset, a.quote.feasible_slack]]
                for a in plan.actions]
    assert got_acts == want["actions"]
    assert [list(c) for c in plan.claims] == want["claims"]
    assert plan.deferred == want["deferred"]
    assert plan.overflow == want["overflow"]
