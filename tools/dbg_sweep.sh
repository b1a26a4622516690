cd /root/repo
for d in ${DBGS:-0 64 0 64 18 80}; do
  ms=$(FW_STEP2D_DBG=$d FW_LIBRARY=$PWD/paper_2311_13049_b200/lib/libfw_b200_exp.so python bench.py --no-cpu-baseline --steps 100 --warmup 5 2>/dev/null | tail -1 | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_step"]*1000,1))')
  echo "dbg=$d: $ms"
done
