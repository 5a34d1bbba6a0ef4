"""Parity on every configuration bench.py measures (VERDICT r1 'pin parity on
every config you benchmark'):

* BASELINE config 4: all 8 shards of the 8 x 65,536-request trace, exactly as
  bench.make_trace builds them (device-drawn trace, GPU), first 60 steps,
  device vs the oracle; shards 1 and 7 also vs the unmodified reference's
  golden logs directly.
* BASELINE config 5: the 200-request long-output trace of the decode leg, a
  full run with the Llama-2-70B KV data plane on, vs the reference's golden
  (event digest, outcomes, MetricsReport) and KV integrity at the end.
* The decode at the benchmarked Llama-2-70B layout (8 KV heads x 8 query heads
  each, split 512, contexts >= 1.5K) vs the fp32/fp64 reference.
* Device MetricsReport (co_metrics) vs the reference's own report on every
  full-run golden fixture.
"""
import hashlib

import numpy as np
import pytest

from tests import golden_io as G
from tests.kv_reference import decode_reference, decode_reference_torch


def test_torch_decode_reference_equals_numpy():
    for rid, ctx, step, L, hq, hkv in [(7, 100, 3, 2, 16, 2), (123456, 37, 99, 1, 8, 8), (5, 300, 1000, 2, 64, 8)]:
        a = decode_reference(rid, ctx, step, L, hq, hkv)
        b = decode_reference_torch(rid, ctx, step, L, hq, hkv, device="cpu")
        assert np.abs(a - b).max() < 1e-12


def _vs_golden(eng, doc, label):
    """Device engine vs a reference golden fixture (oracle/make_golden.py)."""
    from tests.cases import final_arrays
    blob = G.jsonl_bytes(eng.events)
    assert hashlib.sha256(blob).hexdigest() == doc["events_sha256"], f"{label}: event log differs from the reference"
    fd = final_arrays(eng)
    keys = {"generated": "generated", "preemption_count": "preemption_count",
            "preemption_time_us": "preemption_time_us", "max_tbt_us": "max_tbt_us", "kv_need": "kv_need",
            "prefill_done": "prefill_done", "used": "used", "completion_us": "completion_us",
            "first_token_at_us": "first_token_at_us"}
    for ref_key, k in keys.items():
        assert np.array_equal(fd[k], np.asarray(doc["final"][ref_key])), f"{label}: {ref_key}"
    s = eng._scalars()
    assert (s.footprint_tokens, s.used_tokens, s.reserved_blocks_current) == (
        doc["pool"]["footprint"], doc["pool"]["used"], doc["pool"]["reserved"]), label
    samples = [list(x) for x in eng.samples]
    assert hashlib.sha256(__import__("json").dumps(samples).encode()).hexdigest() == doc["samples_sha256"], label


@pytest.fixture(scope="module")
def config4_host_trace():
    import bench
    import paper_2503_13773_b200 as P
    spec = P.PRESETS["sharegpt"].sized(8 * bench.N_PER_GPU, 8e6)
    reqs = P.generate(spec, 0)
    P.assign_slos(reqs, 2_000_000, 200_000, P.SloPolicy(), 0)
    return reqs


@pytest.mark.gpu
@pytest.mark.parametrize("rank", range(8))
def test_config4_shard_first_60_steps(cuda_ok, rank, config4_host_trace):
    import bench
    from oracle.cacheopt_oracle import CacheOptOracle
    from paper_2503_13773_b200 import Engine
    from tests.test_device_parity import _compare
    shard, cfg = bench.make_trace(rank, 8, device=0)   # what the bench runs (device-drawn trace)
    host = config4_host_trace[rank * bench.N_PER_GPU:(rank + 1) * bench.N_PER_GPU]
    assert [(r.id, r.arrival_us, r.prompt_len, r.true_output_len, r.slo_ttft_us, r.slo_tbt_us) for r in shard] == \
        [(r.id, r.arrival_us, r.prompt_len, r.true_output_len, r.slo_ttft_us, r.slo_tbt_us) for r in host]
    eng = Engine(shard, cfg)
    eng.run_steps(60)
    orc = CacheOptOracle(shard, cfg)
    for _ in range(60):
        orc.step()
    _compare(eng, orc, f"config4 shard {rank}")
    name = f"config4_shard{rank}_60"
    if name in G.names():
        _vs_golden(eng, G.load(name), name)
    eng.close()


@pytest.mark.gpu
def test_config2_window_vs_reference_golden(cuda_ok):
    """The bench's own config-2 trace (device-drawn) over the golden window."""
    import bench
    from paper_2503_13773_b200 import Engine
    reqs, cfg = bench.make_trace(0, 1, device=0)
    eng = Engine(reqs, cfg)
    eng.run_steps(60)
    _vs_golden(eng, G.load("config2_60"), "config2_60")
    eng.close()


@pytest.mark.gpu
def test_config5_full_run_with_70b_data_plane(cuda_ok):
    import bench
    import paper_2503_13773_b200 as P
    doc = G.load("config5")
    reqs = bench.long_output_trace()
    greqs, gcfg = G.requests_from(doc)
    assert [(r.id, r.arrival_us, r.prompt_len, r.true_output_len, r.slo_ttft_us, r.slo_tbt_us) for r in reqs] == \
        [(r.id, r.arrival_us, r.prompt_len, r.true_output_len, r.slo_ttft_us, r.slo_tbt_us) for r in greqs]
    kv = P.KVLayout.llama2_70b(host_swap_pages=4096, decode=False)
    eng = P.Engine(reqs, gcfg, kv=kv, steps_per_launch=64)
    bad = checked = 0
    while eng.run_steps(5000) == 5000:  # every live holder's KV checked every 5,000 steps
        b, c = eng.kv_verify()
        bad, checked = bad + b, checked + c
    rep = eng.run()
    _vs_golden(eng, doc, "config5")
    assert rep.to_dict() == doc["metrics"]
    assert bad == 0 and checked > 0
    eng.close()


@pytest.mark.gpu
@pytest.mark.parametrize("name", [n for n in G.names() if n.startswith(("case", "base_", "inv_", "stack_", "config1", "config3"))])
def test_device_metrics_equal_reference_report(cuda_ok, name):
    """Row (f).1 pinned to the reference: Engine.run()'s device-aggregated
    MetricsReport equals the unmodified reference's eng.run().to_dict()."""
    from paper_2503_13773_b200 import Engine
    doc = G.load(name)
    if doc.get("metrics") is None:
        pytest.skip("window fixture")
    reqs, cfg = G.requests_from(doc)
    eng = Engine(reqs, cfg, steps_per_launch=64)
    rep = eng.run()
    assert rep.to_dict() == doc["metrics"], name
    # and the drop-in request states after run() (core.py:113-130)
    done = sum(1 for r in eng.requests.values() if r.state.name == "COMPLETED")
    assert done == doc["metrics"]["completed"]
    eng.close()


def _decode_engine(layers, warm_steps, split=512):
    import bench
    import paper_2503_13773_b200 as P
    kv = P.KVLayout(layers=layers, kv_heads=8, q_heads=64, host_swap_pages=2048, decode=True, decode_split=split)
    cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16),
                         record_events=False)
    eng = P.Engine(bench.long_output_trace(), cfg, kv=kv)
    eng.set_decode(False)
    eng.run_steps(warm_steps)
    eng.set_decode(True)
    return eng


@pytest.mark.gpu
def test_decode_llama2_70b_layout_g8(cuda_ok):
    """G = 8 query heads per KV head, 8 KV heads, split 512, 4 layers, every
    member checked for 6 consecutive decode steps at contexts >= 1.5K."""
    eng = _decode_engine(layers=4, warm_steps=4000)
    checked, long_ctx = 0, 0
    for _ in range(6):
        assert eng.step()
        rids, ctx, out, step_id = eng.last_decode()
        assert len(rids) >= 3
        for k in range(len(rids)):
            ref = decode_reference_torch(rids[k], int(ctx[k]), step_id, 4, 64, 8)
            err = np.abs(out[k] - ref).max() / max(np.abs(ref).max(), 1e-6)
            assert err <= 1e-2, f"member {rids[k]} ctx {ctx[k]}: rel err {err}"
            checked += 1
            long_ctx += int(ctx[k]) >= 1500
    assert checked >= 18 and long_ctx >= 6
    eng.close()


@pytest.mark.gpu
def test_decode_full_80_layer_layout(cuda_ok):
    """The exact benchmarked layout (KVLayout.llama2_70b: 80 layers, 64 q / 8
    kv heads, split 512): 3 decode steps, every member vs the reference."""
    import bench
    import paper_2503_13773_b200 as P
    kv = P.KVLayout.llama2_70b(host_swap_pages=512, decode=True, decode_split=512)
    cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16),
                         record_events=False)
    eng = P.Engine(bench.long_output_trace(), cfg, kv=kv)
    eng.set_decode(False)
    eng.run_steps(3000)
    eng.set_decode(True)
    worst = 0.0
    for _ in range(3):
        assert eng.step()
        rids, ctx, out, step_id = eng.last_decode()
        assert len(rids) >= 3 and int(ctx.max()) >= 1500
        for k in range(len(rids)):
            ref = decode_reference_torch(rids[k], int(ctx[k]), step_id, 80, 64, 8)
            err = np.abs(out[k] - ref).max() / max(np.abs(ref).max(), 1e-6)
            worst = max(worst, err)
    assert worst <= 1e-2, worst
    eng.close()
