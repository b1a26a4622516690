#!/bin/bash
# One GPU call producing the round's measurement evidence (run from the repo root under gpurun).
R=${1:-r1}
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/${R}_bench.json 2> gpurun_out/${R}_bench.err
timeout 600 python bench.py --impl reference > gpurun_out/${R}_bench_ref.json 2> gpurun_out/${R}_bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${R}_launches.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${R}_ncu_launches.log 2>&1
# one step per launch for the full capture, so that its DRAM traffic is per step
FW_STEPS_PER_LAUNCH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_step2d -s 6 -c 1 \
  -o gpurun_out/${R}_prof python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/${R}_ncu_full.log 2>&1
nproc > gpurun_out/${R}_host.txt; lscpu | grep -i "model name" >> gpurun_out/${R}_host.txt
