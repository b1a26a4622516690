cd /root/repo
timeout 300 python bench.py --steps 200 --warmup 5 > gpurun_out/s2_bench.json 2> gpurun_out/s2_bench.err
tail -c 600 gpurun_out/s2_bench.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
echo ncu1 $?
FW_STEPS_PER_LAUNCH=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step2d -s 2 -c 1 -f -o gpurun_out/s2_full python tools/prof_c2.py 4 > gpurun_out/s2_full.log 2>&1
echo ncu2 $?
