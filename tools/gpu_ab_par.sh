# parity subset on the working-tree library, then an A/B of library variants
O=gpurun_out/$1; shift; mkdir -p $O
timeout 900 python -m pytest tests/test_device_parity.py -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
tail -2 $O/pytest.log
bash tools/ab.sh $(basename $O)/ab "$@" | grep -E "==|step" | sed 's/staged.*//'
