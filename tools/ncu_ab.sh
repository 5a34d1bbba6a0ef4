# ncu of k_serial (3rd window step, warm L2, no ncu cache flush) for library
# variants, run under gpurun:  bash tools/ncu_ab.sh <tag> var_a var_b ...
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
for v in "$@"; do
  CACHEOPT_LIB=paper_2503_13773_b200/_lib/$v.so FLUSH=0 timeout 400 ncu --set full --cache-control none \
      --clock-control none -k regex:"^k_serial" -s 42 -c 1 -o $O/$v python tools/step_probe.py ncu > $O/$v.log 2>&1
  ncu -i $O/$v.ncu-rep --page raw --csv > $O/${v}_raw.csv 2>/dev/null
  rm -f $O/$v.ncu-rep
done
