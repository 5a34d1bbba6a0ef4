#!/bin/bash
# Round evidence on one B200 (run under gpurun): bench line, launch list and
# ncu --set full captures of the step's kernels and of the data plane.
# Usage: tools/profile_round.sh [tag]   (outputs under gpurun_out/<tag>/)
set -x
T=${1:-r02}
O=gpurun_out/$T
mkdir -p $O
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 3 --warmup 3 --skip-legs > $O/ncu_launches.log 2>&1
for k in k_serial k_classify; do
  timeout 400 ncu --set full --warp-sampling-interval 0 --clock-control none --import-source on -k regex:"^$k" -s 41 -c 1 \
      -o $O/prof_$k python tools/step_probe.py ncu > $O/ncu_$k.log 2>&1
done
WARM=3000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_decode_tc" -s 3001 -c 1 \
    -o $O/prof_k_decode_tc python tools/decode_once.py decode > $O/ncu_decode.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_data" -c 1 \
    -o $O/prof_k_data python tools/decode_once.py swap > $O/ncu_swap.log 2>&1
python tools/ncu_summary.py $O/prof_*.ncu-rep > $O/ncu_full_summary.csv 2>&1
python tools/launch_summary.py $O/launches.csv > $O/launches_summary.csv 2>&1
for r in $O/prof_*.ncu-rep; do
  ncu -i $r --page details --csv > ${r%.ncu-rep}_details.csv 2>/dev/null
done
ncu -i $O/prof_k_serial.ncu-rep --page source --csv --print-source sass > $O/k_serial_sass.csv 2>/dev/null
# gpurun returns at most 64 MiB: keep the summaries, drop the big reports
find $O -name '*.ncu-rep' -size +6M -delete
ls -la $O
