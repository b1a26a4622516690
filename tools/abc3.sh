#!/bin/bash
# A/B of library variants on the C3 seismic step: tools/abc3.sh main v1 ...
for v in "$@"; do L=""; [ $v != main ] && L=$PWD/paper_2311_13049_b200/lib/libfw_b200_$v.so
FW_LIBRARY=$L python bench.py --workload c3 --steps 10 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', '$v', round(d['ms_per_step'],3), round(d['value'],1))"
done
