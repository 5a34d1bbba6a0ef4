#!/bin/bash
# Round evidence on one B200 (run under gpurun): tests, bench line, phase
# profile, launch list and ncu --set full captures of the top kernels.
# Usage: tools/profile_round.sh [tag]   (outputs under gpurun_out/<tag>/)
set -x
T=${1:-r01}
O=gpurun_out/$T
mkdir -p $O
[ -n "$SKIP_TESTS" ] || timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err
FLUSH_L2=1 timeout 300 python tools/phase_profile.py > $O/phase_profile.txt 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --skip-legs > $O/ncu_launches.log 2>&1
for k in k_plan k_apply k_classify k_bins k_scatter k_begin; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 42 -c 1 \
      -o $O/prof_$k python bench.py --steps 10 --warmup 5 --skip-legs > $O/ncu_$k.log 2>&1
done
if [ -z "$SKIP_LEGS" ]; then
WARM=3000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_decode_tc" -s 3001 -c 1 \
    -o $O/prof_k_decode_tc python tools/decode_once.py decode > $O/ncu_decode.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_data" -c 1 \
    -o $O/prof_k_data python tools/decode_once.py swap > $O/ncu_swap.log 2>&1
fi
python tools/ncu_summary.py $O/prof_*.ncu-rep > $O/ncu_full_summary.csv 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.csv 2>&1
for r in $O/prof_*.ncu-rep; do
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>/dev/null
done
timeout 300 ncu --set full --clock-control none -k regex:"k_arrivals|k_orbit_spec|k_zig_local" -c 3 \
    -o $O/prof_tracegen python tools/tracegen_probe.py > $O/ncu_tracegen.log 2>&1
ncu -i $O/prof_tracegen.ncu-rep --page details --csv > $O/prof_tracegen_details.csv 2>/dev/null
python tools/ncu_summary.py $O/prof_tracegen.ncu-rep > $O/ncu_tracegen_summary.csv 2>&1
# gpurun returns at most 64 MiB: keep the summaries, drop the big reports
find $O -name '*.ncu-rep' -size +6M -delete
ls -la $O
