"""N1/N2/N3 on the device: the KV data plane rides on the block tables.
Every holder's KV must carry its synthetic content after every step (so no
swap-out/in, guest move or fill ever lost or misplaced a byte), the decode
must match an fp32 reference within 1e-2 relative, and switching the data
plane on must not change a single scheduling decision."""
import numpy as np
import pytest

from oracle.cacheopt_oracle import CacheOptOracle
from tests.cases import build_product, case_params
from tests.kv_reference import decode_reference

pytestmark = pytest.mark.gpu

SMALL = dict(layers=2, kv_heads=2, q_heads=4)


def _engine(seed, decode=True, layout=SMALL, split=64):
    import paper_2503_13773_b200 as P
    reqs, cfg = build_product(case_params(seed))
    pages = cfg.capacity_tokens // cfg.sched.small_block_b
    kv = P.KVLayout(**layout, host_swap_pages=16 * pages + 64, decode=decode, decode_split=split)
    return P.Engine(reqs, cfg, kv=kv), reqs, cfg


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 5, 6, 9, 13])
def test_kv_integrity_every_step_and_decisions_unchanged(cuda_ok, seed):
    eng, reqs, cfg = _engine(seed, decode=False)
    orc = CacheOptOracle(reqs, cfg)
    steps = 0
    while True:
        more = eng.step()
        orc.step()
        bad, checked = eng.kv_verify()
        assert bad == 0, f"seed {seed} step {steps}: {bad} of {checked} KV elements wrong"
        steps += 1
        if not more:
            break
    assert eng.events == orc.events
    assert eng.block_tables() == orc.block_tables()
    st = eng.data_stats()
    assert st["fill_bytes"] > 0


def test_swaps_really_move_bytes(cuda_ok):
    # seeds whose truth costs put s* inside the trace's lengths swap a lot
    moved = 0
    for seed in (1, 2, 5, 6):
        if case_params(seed)["truth"] is None:
            continue
        eng, _, _ = _engine(seed, decode=False)
        eng.run_steps(0)
        st = eng.data_stats()
        moved += st["swap_out_bytes"] + st["swap_in_bytes"]
    assert moved > 0


# (seed, layout, split): G = 2 and G = 16 query heads per KV head (the
# tcgen05 kernel's 8- and 16-head softmax variants), splits shorter and
# longer than its 128-position tile
DECODE_CASES = [(1, SMALL, 64), (5, SMALL, 64), (2, dict(layers=1, kv_heads=1, q_heads=16), 300),
                (6, dict(layers=2, kv_heads=2, q_heads=16), 512)]


@pytest.mark.parametrize("seed,layout,split", DECODE_CASES)
def test_decode_matches_fp32_reference(cuda_ok, seed, layout, split):
    eng, _, _ = _engine(seed, decode=True, layout=layout, split=split)
    checked = 0
    for _ in range(400):
        if not eng.step():
            break
        rids, ctx, out, step_id = eng.last_decode()
        for k in range(0, len(rids), max(1, len(rids) // 3)):
            ref = decode_reference(rids[k], int(ctx[k]), step_id, layout["layers"], layout["q_heads"],
                                   layout["kv_heads"])
            err = np.abs(out[k] - ref).max() / max(np.abs(ref).max(), 1e-6)
            assert err <= 1e-2, f"member {rids[k]} ctx {ctx[k]}: rel err {err}"
            checked += 1
    assert checked > 20


@pytest.mark.parametrize("seed", [8, 27, 65, 139])
def test_kv_integrity_with_stacked_guests(cuda_ok, seed):
    # a host release re-homes several guests at once: the earlier guests' new
    # pages may be the pages holding a later guest's KV (staged as one group)
    import paper_2503_13773_b200 as P
    p = case_params(seed)
    p["allow_stacking"] = True
    reqs, cfg = build_product(p)
    pages = cfg.capacity_tokens // cfg.sched.small_block_b
    kv = P.KVLayout(**SMALL, host_swap_pages=16 * pages + 64, decode=False)
    eng = P.Engine(reqs, cfg, kv=kv)
    orc = CacheOptOracle(reqs, cfg)
    while True:
        more = eng.step()
        orc.step()
        bad, checked = eng.kv_verify()
        assert bad == 0, f"seed {seed}: {bad} of {checked} KV elements wrong"
        if not more:
            break
    assert eng.events == orc.events
    assert eng.block_tables() == orc.block_tables()
    if getattr(orc, "multi_rehomes", 0):  # 27, 65, 139: host releases re-home 2+ guests at once
        assert eng.data_stats()["move_bytes"] > 0
