#!/bin/bash
# Round-2 evidence of the multi-pass configurations (run from the repo root under gpurun):
# bench lines of C3 / C4 / C5, ncu launch lists of C5 and C3, full captures of C5's two big kernels.
R=${1:-r2b}
mkdir -p gpurun_out
for w in c3 c4 c5; do
  timeout 600 python bench.py --workload $w > gpurun_out/${R}_bench_$w.json 2> gpurun_out/${R}_bench_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_c5_launches.csv \
  python tools/c5batch.py > gpurun_out/${R}_c5_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_c3_launches.csv \
  python bench.py --workload c3 --steps 2 --warmup 1 > gpurun_out/${R}_c3_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lines_terms -s 1 -c 1 -f \
  -o gpurun_out/${R}_c5_lt python tools/c5batch.py > gpurun_out/${R}_c5_lt.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows_c2r -s 1 -c 1 -f \
  -o gpurun_out/${R}_c5_c2r python tools/c5batch.py > gpurun_out/${R}_c5_c2r.log 2>&1
