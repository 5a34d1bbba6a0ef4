# compute-sanitizer memcheck / racecheck / synccheck over small regimes (run
# under gpurun); logs under gpurun_out/<tag>/ (copied to profiles/ by hand)
T=${1:-san}; O=gpurun_out/$T; mkdir -p $O
for tool in memcheck racecheck synccheck; do
  for m in sched data; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
        python tools/sanitize_case.py $m 1 > $O/${tool}_${m}.log 2>&1
    echo "$tool $m rc=$?" >> $O/summary.txt
    tail -3 $O/${tool}_${m}.log >> $O/summary.txt
  done
done
cat $O/summary.txt
