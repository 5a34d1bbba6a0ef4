# Development iteration on one B200: quick parity subset, step timing, and an
# ncu source-level capture of the step's serial kernel.
# Usage (under gpurun): bash tools/gpu_iter.sh <tag> [full]
T=${1:-it}; O=gpurun_out/$T; mkdir -p $O
if [ "$2" = "full" ]; then
  timeout 900 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1
else
  timeout 600 python -m pytest tests/test_device_parity.py tests/test_baselines.py tests/test_multi_instance.py -m gpu -q -x > $O/pytest.log 2>&1
fi
echo "pytest rc=$?" >> $O/pytest.log
timeout 200 python tools/step_probe.py time > $O/step_probe.txt 2>&1
timeout 600 ncu --set full --warp-sampling-interval 0 --clock-control none --cache-control none --import-source on -k regex:"k_serial" -s 41 -c 1 -o $O/k_serial python tools/step_probe.py ncu > $O/ncu_k_serial.log 2>&1
ncu -i $O/k_serial.ncu-rep --page source --csv --print-source sass > $O/k_serial_sass.csv 2>/dev/null
ncu -i $O/k_serial.ncu-rep --page details --csv > $O/k_serial_details.csv 2>/dev/null
find $O -name '*.ncu-rep' -size +40M -delete
tail -2 $O/pytest.log; cat $O/step_probe.txt
