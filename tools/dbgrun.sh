for d in 0 1 2 4 8 15; do
  FW_STEP2D_DBG=$d timeout 120 python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dbg', $d, round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1
done
