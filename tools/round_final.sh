#!/bin/bash
# Final evidence of the round (run from the repo root under gpurun): the C2 bench line and its
# reference arm, the ncu launch list of the same command, one full capture of k_step2d (one step
# per launch so that its DRAM traffic is per step), then the multi-pass configurations.
R=${1:-r2f}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${R}_bench_c2.json 2> gpurun_out/${R}_bench_c2.err
timeout 900 python bench.py --impl reference > gpurun_out/${R}_bench_c2_reference.json 2> gpurun_out/${R}_bench_c2_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${R}_c2_launches.csv \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_c2_ncu_launches.log 2>&1
FW_STEPS_PER_LAUNCH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step2d -s 4 -c 1 -f \
  -o gpurun_out/${R}_c2_full python tools/prof_c2.py 4 > gpurun_out/${R}_c2_full.log 2>&1
tools/round_evidence2.sh ${R}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${R}_c4_launches.csv \
  python bench.py --workload c4 --steps 1 --warmup 1 > gpurun_out/${R}_c4_ncu.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rows_c2r -s 1 -c 1 -f \
  -o gpurun_out/${R}_c3_c2r python bench.py --workload c3 --steps 1 --warmup 1 > gpurun_out/${R}_c3_c2r.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_linesILi256 -s 4 -c 1 -f \
  -o gpurun_out/${R}_c3_lines python bench.py --workload c3 --steps 1 --warmup 1 > gpurun_out/${R}_c3_lines.log 2>&1
