#!/bin/bash
# usage: abcfg.sh variant...   (main = in-tree library)
for v in "$@"; do L=""; [ $v != main ] && L=$PWD/paper_2311_13049_b200/lib/libfw_b200_$v.so
FW_LIBRARY=$L python bench.py --workload c5 --steps 40 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5', '$v', {k: round(v['ms_per_sweep'],3) for k,v in d['config']['M_sweep'].items()})"
FW_LIBRARY=$L python bench.py --workload c3 --steps 10 --warmup 2 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', '$v', round(d['ms_per_step'],3), round(d['value'],1))"
done
