O=gpurun_out/$1; mkdir -p $O
timeout 900 python -m pytest tests/test_plan_batch_device.py -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -25 $O/pytest.log
timeout 300 python tools/e2e_gap.py > $O/e2e_gap.txt 2>&1; cat $O/e2e_gap.txt
