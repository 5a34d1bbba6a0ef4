O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_device_parity.py tests/test_reference_engine_cases.py tests/test_data_plane.py tests/test_multi_instance.py -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
timeout 300 python tools/e2e_gap.py > $O/e2e_gap.txt 2>&1; cat $O/e2e_gap.txt
timeout 600 python bench.py --skip-legs > $O/bench.json 2> $O/bench.err
python - <<PY
import json
d = json.load(open("$O/bench.json"))
print("ms_per_step", d["ms_per_step"], "value", d["value"], "e2e", d["e2e"]["value"], "nodrain", d["e2e"].get("without_event_drain"), "cpu", d["cpu_baseline"]["value"])
PY
