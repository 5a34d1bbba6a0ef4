#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): tests, bench line,
# launch list and ncu --set full captures of the top kernels.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --skip-legs > gpurun_out/ncu_launches.log 2>&1
for k in k_plan k_apply k_classify k_scatter; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:"^$k" -s 42 -c 1 \
      -o gpurun_out/prof_$k python bench.py --steps 10 --warmup 5 --skip-legs > gpurun_out/ncu_$k.log 2>&1
done
WARM=3000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_decode_tc" -s 3001 -c 1 \
    -o gpurun_out/prof_k_decode_tc python tools/decode_once.py decode > gpurun_out/ncu_decode.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_data" -c 1 \
    -o gpurun_out/prof_k_data python tools/decode_once.py swap > gpurun_out/ncu_swap.log 2>&1
ls -la gpurun_out
