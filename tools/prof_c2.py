"""Profiling driver: C2 seismic steps (configs[1]) through the public stepper, one persistent
launch per step (FW_STEPS_PER_LAUNCH=1), for ncu captures of k_step2d.
usage: python tools/prof_c2.py [steps]   (FW_STEP2D_TM=1 selects the time-multiplexed kernel)"""
import os
import sys

os.environ.setdefault("FW_STEPS_PER_LAUNCH", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_13049_b200 as fw  # noqa: E402
from paper_2311_13049_b200 import configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4
cfg = configs.c2()
g = fw.Grid(list(zip(cfg.lo, cfg.hi)), cfg.J)
st = fw.SeismicStepper(fw.build_medium(g, cfg.gamma, cfg.c0, 1.0, cfg.M), cfg.phi, cfg.psi, cfg.tau)
st.advance(steps)
print("n =", st.n(), "persistent =", st.persistent)
os._exit(0)
