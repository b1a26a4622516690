#!/bin/bash
# Timing experiments of the persistent C2 kernel (wrong results by design): an experiments build
# (tools/variants.sh exp "-DFW_STEP2D_EXPERIMENTS=1") run with FW_STEP2D_DBG=bits, one bench per value.
cd "$(dirname "$0")/.."
for d in ${DBGS:-0 2 4 16 32 48}; do
  ms=$(FW_STEP2D_DBG=$d FW_LIBRARY=$PWD/paper_2311_13049_b200/lib/libfw_b200_exp.so timeout 90 python bench.py --no-cpu-baseline --steps 100 --warmup 5 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')
  echo "dbg=$d: $ms"
done
