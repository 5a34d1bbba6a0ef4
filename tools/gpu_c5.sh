O=gpurun_out/$1; mkdir -p $O
timeout 1500 python tools/config5_run.py 1000 > $O/config5_run.txt 2>&1; tail -4 $O/config5_run.txt
