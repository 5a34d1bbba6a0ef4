# racecheck of the data plane on a short window (the full run exceeds 15 min
# under racecheck): per-step API then one multi-step graph, decode on
T=${1:-san2}; O=gpurun_out/$T; mkdir -p $O
timeout 1500 compute-sanitizer --tool racecheck --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_case.py data 1 20 > $O/racecheck_data.log 2>&1
echo "racecheck data rc=$?" >> $O/summary.txt; tail -3 $O/racecheck_data.log >> $O/summary.txt
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_case.py stack 27 > $O/${tool}_stack.log 2>&1
  echo "$tool stacking+split-io rc=$?" >> $O/summary.txt; tail -3 $O/${tool}_stack.log >> $O/summary.txt
done
cat $O/summary.txt
