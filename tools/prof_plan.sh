set -x
O=gpurun_out/p1; mkdir -p $O
python tools/step_probe.py time > $O/time.txt 2>&1
for k in k_plan k_apply; do
timeout 600 ncu --set full --clock-control none --cache-control none --import-source on -k regex:"^$k" -s 41 -c 1 -o $O/$k python tools/step_probe.py ncu > $O/ncu_$k.log 2>&1
ncu -i $O/$k.ncu-rep --page source --csv --print-source sass > $O/${k}_sass.csv 2>/dev/null
ncu -i $O/$k.ncu-rep --page details --csv > $O/${k}_details.csv 2>/dev/null
done
ls -la $O
