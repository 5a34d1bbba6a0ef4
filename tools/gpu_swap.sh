O=gpurun_out/$1; mkdir -p $O
timeout 1500 python tools/swap_probe.py 500 > $O/swap_probe.txt 2>&1; tail -4 $O/swap_probe.txt
