O=gpurun_out/$1; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -x > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
tail -3 $O/pytest_gpu.log
timeout 300 python tools/step_probe.py time > $O/step_probe.txt 2>&1; cat $O/step_probe.txt
timeout 900 python tools/swap_probe.py 2000 200 24576 > $O/swap_probe.txt 2>&1; tail -4 $O/swap_probe.txt
