O=gpurun_out/$1; mkdir -p $O
timeout 1200 python -m pytest tests/test_pool_device.py tests/test_sched_ops_device.py tests/test_device_parity.py -k "stacking or pool or sched or Pool or allocate or classify or victim or pair or budget or proactive or demand or grow or embed or reserve or release or constructor" -m gpu -q > $O/pytest_new.log 2>&1; echo "rc=$?" >> $O/pytest_new.log
timeout 900 python -m pytest tests/test_data_plane.py -k stacked -m gpu -q > $O/pytest_dp.log 2>&1; echo "rc=$?" >> $O/pytest_dp.log
tail -15 $O/pytest_new.log; tail -5 $O/pytest_dp.log
