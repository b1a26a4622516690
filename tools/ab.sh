#!/bin/bash
# A/B timing of library variants on the GPU box: tools/ab.sh name1 name2 ...  (C2 bench, us/step)
# (extra environment, e.g. FW_STEPS_PER_LAUNCH=1, passes through to every run)
cd "$(dirname "$0")/.."
for rep in 1 2; do
  for v in "$@"; do
    lib=$PWD/paper_2311_13049_b200/lib/libfw_b200_$v.so
    ms=$(FW_LIBRARY=$lib timeout 120 python bench.py --no-cpu-baseline --steps 100 --warmup 5 2>/dev/null | tail -1 |
         python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1), d["clocks"]["sm_mhz"])')
    echo "$v rep$rep: $ms"
  done
done
