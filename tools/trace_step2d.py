"""Run a few C2 steps with FW_TRACE=1 and print the per-warp phase timeline of CTA 0 / CTA 100."""
import ctypes as C
import os
import sys

import numpy as np

os.environ["FW_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_13049_b200 as fw  # noqa: E402
from paper_2311_13049_b200 import configs  # noqa: E402

cfg = configs.c2()
ctx = fw.Context(0)
g = fw.Grid(list(zip(cfg.lo, cfg.hi)), cfg.J)
st = fw.SeismicStepper(fw.build_medium(g, cfg.gamma, cfg.c0, 1.0, cfg.M), cfg.phi, cfg.psi, cfg.tau, ctx=ctx)
st.advance(3)
lib = fw.load_library()
lib.fw_ctx_trace.argtypes = [C.c_void_p, C.c_void_p]
buf = np.zeros(2 * 16 * 136 * 4, dtype=np.uint64)
fw._capi.check(lib.fw_ctx_trace(ctx.handle, buf.ctypes.data))
tr = buf.reshape(2, 16, 136, 4).astype(np.int64)
ntot = 34
t0 = tr[tr > 0].min()
for sel in range(2):
    print(f"=== CTA {0 if sel == 0 else 100} (times in us from first mark)")
    for w in range(16):
        d = tr[sel, w, :ntot]
        if d.max() == 0:
            continue
        d = (d - t0) / 1000.0
        role = "col" if w < 8 else "row"
        waits = d[:, 1] - d[:, 0]
        work1 = d[:, 2] - d[:, 1]
        work2 = d[:, 3] - d[:, 2]
        print(f"w{w:2d} {role} start {d[0,0]:8.1f} end {d[ntot-1,3]:8.1f} | wait mean {waits.mean():6.2f} max {waits.max():6.2f}"
              f" | phaseA mean {work1.mean():6.2f} | phaseB mean {work2.mean():6.2f}")
    w = 0 if sel == 0 else 0
    d = (tr[sel, 0, :8] - t0) / 1000.0
    print("col w0 first terms:", np.round(d, 1).tolist())
    d = (tr[sel, 8, :8] - t0) / 1000.0
    print("row w8 first terms:", np.round(d, 1).tolist())
