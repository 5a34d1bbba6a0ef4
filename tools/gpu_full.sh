# Full GPU test suite + bench (run under gpurun): bash tools/gpu_full.sh <tag> [bench-args]
T=${1:-full}; shift; O=gpurun_out/$T; mkdir -p $O
timeout 1000 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 600 python bench.py "$@" > $O/bench.json 2> $O/bench.err
tail -3 $O/pytest_gpu.log
python - <<PY
import json
d = json.load(open("$O/bench.json"))
print("ms_per_step", d["ms_per_step"], "value", d["value"], "e2e", d["e2e"]["value"], "nodrain", d["e2e"].get("without_event_drain"))
PY
