"""Profile -> fit -> sweet spot on this B200: writes
coefficients.json like the reference's `kvcsim fit` (cli.py:440-447) plus the
measured samples.  python tools/cost_profile.py [13b|70b] [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_13773_b200 import KVLayout, costprofile as cp  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "70b"
kv = KVLayout.llama2_70b(decode=False) if which == "70b" else KVLayout.llama2_13b(decode=False)
dims = cp.ModelDims.llama2_70b() if which == "70b" else cp.ModelDims.llama2_13b()
res = cp.hardware_truth(kv_layout=kv, dims=dims)
res.pop("truth")
res["model"] = dims.name
res["bytes_per_token"] = kv.bytes_per_token
txt = json.dumps(res, indent=1, sort_keys=True)
if len(sys.argv) > 2:
    with open(sys.argv[2], "w") as fh:
        fh.write(txt + "\n")
print(json.dumps({k: res[k] for k in ("model", "swap", "recompute", "sweet_spot", "crossover_note")}))
