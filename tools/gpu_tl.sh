O=gpurun_out/$1; mkdir -p $O
CACHEOPT_LIB=paper_2503_13773_b200/_lib/var_prof.so timeout 300 python tools/phase_timeline.py > $O/timeline.txt 2>&1; cat $O/timeline.txt
