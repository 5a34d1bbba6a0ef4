# A/B step timing of library variants on ONE box (run under gpurun):
#   bash tools/ab.sh <tag> var_a var_b ...   (paper_2503_13773_b200/_lib/<var>.so)
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
for rep in 1 2 3; do
  for v in "$@"; do
    echo "== $v rep $rep" >> $O/ab.txt
    CACHEOPT_LIB=paper_2503_13773_b200/_lib/$v.so timeout 200 python tools/step_probe.py time >> $O/ab.txt 2>&1
  done
done
cat $O/ab.txt
