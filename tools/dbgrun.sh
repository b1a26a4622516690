# needs a library built with FW_BUILD_EXPERIMENTS=1 (python -c "import __graft_entry__ as g; g.build_library(True)")
# timing experiments (FW_STEP2D_DBG bits: 1 no (s-s0)^m loads, 2 no weight loads, 4 no tile TMA,
# 8 one ring slot, 16 rows do pass 0 only, 32 columns skip the FFT); results are wrong by design
for d in ${DBG_LIST:-0 1 2 4 8 15 16 32}; do
  FW_STEP2D_DBG=$d timeout 120 python bench.py --no-cpu-baseline --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('dbg', $d, round(d['ms_per_step']*1000,1), 'us')" 2>&1 | tail -1
done
