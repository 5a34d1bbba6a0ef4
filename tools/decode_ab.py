"""Development aid: the bench decode leg (config 5) with the kernel chosen by
the engine's decode kernel."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

r = bench.decode_leg(0, warm_steps=int(os.environ.get("WARM", "6000")))
print(json.dumps({"tok_s": r["value"],
                  "frac": r["roofline"]["frac"], "gbs": r["roofline"]["achieved"],
                  "ms": r["decode_ms_per_step"], "integrity": r["kv_integrity"]}))
