"""N4 host-side logic on CPU with the gloo backend (world size 2), and the
device all-reduce path on one GPU (a 1-rank communicator)."""
import os
import socket

import pytest
import torch.multiprocessing as mp

from oracle.cacheopt_oracle import CacheOptOracle
from paper_2503_13773_b200.multi import broadcast_uid, reduce_reserve_cpu, shard
from tests.cases import config2


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        reqs, cfg = config2(n=2048, capacity=8_192)
        mine = shard(reqs, rank, world)
        uid = broadcast_uid(bytes(range(128)) if rank == 0 else bytes(128))
        orc = CacheOptOracle(mine, cfg)
        totals = []
        for _ in range(25):
            orc.step()
            totals.append(reduce_reserve_cpu(orc.free_tokens(), orc.rsv_cur))
        out[rank] = (uid, [r.id for r in mine], totals, len(orc.events))
    finally:
        dist.destroy_process_group()


def test_two_instances_gloo_reserve_totals():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    uid0, ids0, tot0, _ = out[0]
    uid1, ids1, tot1, _ = out[1]
    assert uid0 == uid1 == bytes(range(128))
    assert not set(ids0) & set(ids1) and len(ids0) + len(ids1) == 2048
    assert tot0 == tot1
    # the all-reduced totals equal the sum of the two independent instances
    reqs, cfg = config2(n=2048, capacity=8_192)
    a, b = (CacheOptOracle(shard(reqs, r, world), cfg) for r in range(world))
    for k in range(25):
        a.step(); b.step()
        assert tot0[k] == (a.free_tokens() + b.free_tokens(), a.rsv_cur + b.rsv_cur)


def test_shards_are_contiguous_and_disjoint():
    reqs, _ = config2(n=1000, capacity=8_192)
    parts = [shard(reqs, r, 8) for r in range(8)]
    flat = [r.id for p in parts for r in p]
    assert flat == list(range(1000))
    with pytest.raises(ValueError):
        shard(reqs, 8, 8)


@pytest.mark.gpu
def test_one_rank_nccl_reserve_matches_instance(cuda_ok):
    from paper_2503_13773_b200 import Engine
    from paper_2503_13773_b200.multi import attach_global_reserve
    from tests.cases import build_product, case_params
    reqs, cfg = build_product(case_params(3))
    eng = Engine(reqs, cfg)
    attach_global_reserve(eng, 0, 1)
    orc = CacheOptOracle(reqs, cfg)
    for _ in range(30):
        eng.step()
        orc.step()
        free, rsv, _ = eng.global_reserve()
        assert (free, rsv) == (orc.free_tokens(), orc.rsv_cur)
    eng.run_steps(200)
    for _ in range(200):
        orc.step()
    assert eng.events == orc.events  # telemetry never changes a decision
    # the multi-step graph's deferred joins: the last slot holds the last step's totals
    assert eng.global_reserve()[:2] == (orc.free_tokens(), orc.rsv_cur)
    assert eng.global_reserve()[2] > 0


@pytest.mark.gpu
def test_collective_mode_runs_fixed_step_counts_past_the_end(cuda_ok):
    # with a communicator every rank must enqueue the same number of steps even
    # after its own shard finished (an early-finishing rank must not hang others)
    from paper_2503_13773_b200 import Engine
    from paper_2503_13773_b200.multi import attach_global_reserve
    from tests.cases import build_product, case_params
    reqs, cfg = build_product(case_params(2))
    eng = Engine(reqs, cfg, steps_per_launch=16)
    orc = CacheOptOracle(reqs, cfg)
    total = orc.run()
    attach_global_reserve(eng, 0, 1)
    eng.run_steps(total + 100)
    free, rsv, calls = eng.global_reserve()
    assert calls >= total + 100
    assert (free, rsv) == (orc.free_tokens(), orc.rsv_cur)
    assert eng.events == orc.events
    assert eng.step_result()[0] is False  # finished, and still enqueues its collective
