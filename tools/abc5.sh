#!/bin/bash
# A/B of library variants on C5 (M sweep) and the C2 multi-pass step: tools/abc5.sh main v1 ...
for v in "$@"; do L=""; [ $v != main ] && L=$PWD/paper_2311_13049_b200/lib/libfw_b200_$v.so
FW_LIBRARY=$L python bench.py --workload c5 --steps 40 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', '$v', {k: round(v['ms_per_sweep'],3) for k,v in d['config']['M_sweep'].items()})"
done
