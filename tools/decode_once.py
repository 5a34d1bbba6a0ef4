"""Profiling driver: build a decode-heavy state (config 5 layout) and run a
few steps with decode on, so ncu can capture k_decode_tc / k_data."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2503_13773_b200 as P  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "decode"
if mode == "swap":
    kv = P.KVLayout.llama2_70b(host_swap_pages=320, decode=False)
    cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16))
    eng = P.Engine(bench.long_output_trace(n=8), cfg, device=0, kv=kv)
    print(eng.swap_bench(4731, iters=2))
else:
    kv = P.KVLayout.llama2_70b(host_swap_pages=4096, decode=True, decode_split=512)
    cfg = P.EngineConfig(capacity_tokens=65_536, reserved_blocks=8, sched=P.SchedulerConfig(small_block_b=16),
                         record_events=False)
    eng = P.Engine(bench.long_output_trace(), cfg, device=0, kv=kv)
    eng.set_decode(False)
    eng.run_steps(int(os.environ.get("WARM", "3000")))
    eng.set_decode(True)
    for _ in range(3):
        eng.step()
    print(eng.data_stats())
