for spl in ${SPL_LIST:-1 0}; do
  FW_STEPS_PER_LAUNCH=$spl timeout 120 python bench.py --no-cpu-baseline --steps 100 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('steps/launch', $spl, round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1
done
