#!/bin/bash
# A/B of library variants on C4 (one seismic step after one warm-up): tools/abc4.sh main v1 ...
for v in "$@"; do L=""; [ $v != main ] && L=$PWD/paper_2311_13049_b200/lib/libfw_b200_$v.so
FW_LIBRARY=$L python bench.py --workload c4 --steps 2 --warmup 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c4', '$v', round(d['ms_per_step'],2), round(d['value'],1))"
done
