O=gpurun_out/$1; mkdir -p $O
timeout 1500 python -m pytest tests/test_data_plane.py tests/test_bench_configs.py tests/test_costprofile.py -m gpu -q -x > $O/pytest_dp.log 2>&1; echo "rc=$?" >> $O/pytest_dp.log
tail -5 $O/pytest_dp.log
timeout 900 python tools/swap_probe.py 3000 50 > $O/swap_probe.txt 2>&1; cat $O/swap_probe.txt | tail -8
