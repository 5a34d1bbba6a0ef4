import sys; sys.path.insert(0, '.')
import paper_2503_13773_b200 as P
from tests.cases import build_product, case_params
from oracle.cacheopt_oracle import CacheOptOracle
seed = int(sys.argv[1])
reqs, cfg = build_product(case_params(seed))
pages = cfg.capacity_tokens // cfg.sched.small_block_b
for hp in (16 * pages + 64, 256 * pages):
    kv = P.KVLayout(layers=2, kv_heads=2, q_heads=4, host_swap_pages=hp, decode=False, decode_split=64)
    eng = P.Engine(reqs, cfg, kv=kv)
    orc = CacheOptOracle(reqs, cfg)
    n = 0
    try:
        while True:
            more = eng.step(); orc.step(); n += 1
            if n % 50 == 0 or not more:
                ev_d, ev_o = eng.events, orc.events
                if ev_d != ev_o:
                    k = next((k for k, (a, b) in enumerate(zip(ev_d, ev_o)) if a != b), min(len(ev_d), len(ev_o)))
                    print("hp", hp, "step", n, "DIFF at event", k, ev_d[k:k+2], ev_o[k:k+2]); break
            if not more:
                print("hp", hp, "ok", n, eng.data_stats()); break
    except Exception as e:
        print("hp", hp, "step", n, "EXC", e)
