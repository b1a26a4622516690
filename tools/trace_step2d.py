"""(Needs a library built with FW_BUILD_TRACE=1 python -c "import __graft_entry__ as g; g.build_library(True)".)
Run a few C2 steps with FW_TRACE=1 and print the per-warp phase timeline of CTA 0 / CTA 100
of the persistent step kernel (fw_step2d.cu, FW_TRACE marks; 8 marks per warp and term).

column warps: 0 term start | 1 weights + uhat loaded | 2 ring slot free | 3 pass 0 | 4 pass 1
              | 5 pass 2 + pre-processing + Z stores | 6 group barrier
row warps:    0 term start | 2 tile of Z[t] landed (TMA) | 4 pass 0 + tile released | 5 pass 1
              | 6 pass 2 + recombination | 7 pair barrier
"""
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
st.advance(6)
lib = fw.load_library()
lib.fw_ctx_trace.argtypes = [C.c_void_p, C.c_void_p]
buf = np.zeros(2 * 32 * 136 * 8 + 2 * 160 * 2 * 136, dtype=np.uint64)
fw._capi.check(lib.fw_ctx_trace(ctx.handle, buf.ctypes.data))
tr = buf[:2 * 32 * 136 * 8].reshape(2, 32, 136, 8).astype(np.int64)
colend = buf[2 * 32 * 136 * 8:2 * 32 * 136 * 8 + 160 * 2 * 136].reshape(160, 2, 136).astype(np.int64)
colgo = buf[2 * 32 * 136 * 8 + 160 * 2 * 136:].reshape(160, 2, 136).astype(np.int64)  # after the ring wait
ntot = 34
# warp roles (fw_step2d.cu): FW_TRACE_LAYOUT=w16 -> rows 0-6, agents 7, columns 8-15
LAYOUT = os.environ.get("FW_TRACE_LAYOUT", "w24")
COLW0, ROWW0, PRODW = {"w16": (8, 0, 7), "w20": (12, 0, 8)}.get(LAYOUT, (16, 0, 14))
t0 = tr[:, :24][tr[:, :24] > 0].min()
COL = ["w+uhat", "ring", "pass0", "pass1", "pass2+Z", "gbar"]
ROW = ["tile wait", "pass0", "pass1", "pass2+acc", "pairbar"]
ROWMARKS = [0, 2, 4, 5, 6, 7]
for sel in range(2):
    print(f"=== CTA {0 if sel == 0 else 100} (us; mean per term over terms 2..{ntot - 1})")
    for w in range(24):
        d = tr[sel, w, :ntot]
        if d.max() == 0:
            continue
        iscol = COLW0 <= w < COLW0 + 8
        names = COL if iscol else ROW
        nm = len(names) + 1
        d = (d[:, :nm] if iscol else d[:, ROWMARKS]).astype(np.float64)
        ok = (d > 0).all(axis=1)
        d = (d - t0) / 1000.0
        rng = [i for i in range(2, ntot) if ok[i]]
        if not rng:
            print(f"w{w:2d} (inactive)")
            continue
        dd = d[rng]
        per = np.diff(dd, axis=1).mean(axis=0)
        nxt = [d[i + 1, 0] - d[i, 0] for i in rng if i + 1 < ntot and ok[i + 1]]
        print(f"w{w:2d} {'col' if iscol else 'row'} term {np.mean(nxt) if nxt else float('nan'):5.2f} | "
              + " ".join(f"{n} {x:5.2f}" for n, x in zip(names, per))
              + f" | start {d[0, 0]:6.1f} end {d[ntot - 1, nm - 1]:6.1f}")

# launch marks: warp slot 31, [step % 64][entry, exit] (CTA 0)
lm = buf[:2 * 32 * 136 * 8].reshape(2, 32, 136 * 8)[0, 31, :128].reshape(64, 2).astype(np.int64)
ok = np.nonzero(lm[:, 0] > 0)[0]
if len(ok):
    print("launch marks (CTA 0, us): step: entry -> exit (duration), gap from previous exit")
    prev = None
    for k in sorted(ok, key=lambda i: lm[i, 0]):
        e0, e1 = lm[k]
        gap = (e0 - prev) / 1000.0 if prev is not None else float("nan")
        print(f"  slot {k:2d}: {(e1 - e0) / 1000.0:8.1f} us, gap {gap:6.1f} us; first term mark at "
              f"{(tr[0, :24][tr[0, :24] > 0].min() - e0) / 1000.0 if k == ok[-1] else float('nan'):6.1f}")
        prev = e1

# step start marks (term slot 135): columns [0] before the F1 wait, [1] F1 complete, [2] F2 complete;
# rows [0] F1 start, [1] F1 signalled
for sel in range(2):
    c = (tr[sel, COLW0, 135, :4] - t0) / 1000.0
    r = (tr[sel, ROWW0, 135, :7] - t0) / 1000.0
    lt = (tr[sel, ROWW0, ntot - 1, :8] - t0) / 1000.0
    f = (tr[sel, COLW0, 0, 0] - t0) / 1000.0
    print(f"CTA {0 if sel == 0 else 100}: rows F1 {r[0]:.1f} -> {r[1]:.1f} us; columns wait F1 {c[0]:.1f} -> {c[1]:.1f},"
          f" F2 passes done {c[3]:.1f}, F2 done {c[2]:.1f}, first term starts {f:.1f} us (t0 = earliest mark)")
    print(f"  rows' last term: start {lt[0]:.1f}, tile {lt[2]:.1f}, pass 2 done {lt[6]:.1f}, pairbar {lt[7]:.1f};"
          f" update start {r[6]:.1f} done {r[2]:.1f} us")

# producer (row warp 14, lane 0): [0] loop top, [1] cC[t] complete, [2] tile_empty(t-1), [3] TMA issued;
# consumers (row warp 0): [0] term start, [2] tile landed; columns (first column warp): [6] term done
for sel in range(2):
    P = (tr[sel, PRODW, :ntot, :4] - t0) / 1000.0
    R = (tr[sel, ROWW0, :ntot, :8] - t0) / 1000.0
    Cw = (tr[sel, COLW0, :ntot, :8] - t0) / 1000.0
    print(f"CTA {0 if sel == 0 else 100}: t | cols done | cC ready | empty(t-1) | TMA issue | landed | row wants")
    for t in range(1, ntot):
        print(f"  {t:2d} | {Cw[t, 6]:7.1f} | {P[t, 1]:7.1f} | {P[t, 2]:7.1f} | {P[t, 3]:7.1f} | {R[t, 2]:7.1f} | {R[t, 0]:7.1f}")

# every CTA's column groups: mean term duration (terms 2..ntot-1) and finishing time of the last term
ce = colend[:148, :, :ntot]
act = (ce > 0).all(axis=2)
dur = np.where(act, (ce[:, :, ntot - 1] - ce[:, :, 1]) / 1000.0 / (ntot - 2), np.nan)
fin = np.where(act, (ce[:, :, ntot - 1] - t0) / 1000.0, np.nan)
print("column groups: mean us/term (terms 2..): min %.2f median %.2f max %.2f" % (np.nanmin(dur), np.nanmedian(dur), np.nanmax(dur)))
order = np.argsort(-np.nan_to_num(dur, nan=-1).ravel())[:12]
print("slowest groups (cta, group, us/term, last term done):",
      [(int(i // 2), int(i % 2), round(float(dur.ravel()[i]), 2), round(float(fin.ravel()[i]), 1)) for i in order])
ng = act.sum(axis=1)
for k in (1, 2):
    sel = ng == k
    if sel.any():
        print(f"CTAs with {k} active group(s): {int(sel.sum())}, mean us/term {np.nanmean(dur[sel]):.2f}")

# own work per term (ring wait excluded) = term end - after-ring-wait, terms 2..ntot-1
cg_ = colgo[:148, :, :ntot]
own = np.where(act, (ce[:, :, 2:ntot] - cg_[:, :, 2:ntot]).mean(axis=2) / 1000.0, np.nan)
print("own column work us/term: min %.2f median %.2f max %.2f" % (np.nanmin(own), np.nanmedian(own), np.nanmax(own)))
order = np.argsort(-np.nan_to_num(own, nan=-1).ravel())[:16]
print("largest own work (cta, group, us):", [(int(i // 2), int(i % 2), round(float(own.ravel()[i]), 2)) for i in order])
for k in (1, 2):
    sel = ng == k
    if sel.any():
        print(f"CTAs with {k} group(s): own work mean {np.nanmean(own[sel]):.2f} max {np.nanmax(own[sel]):.2f}")
nrows = np.array([((b + 1) * 1024) // 148 - (b * 1024) // 148 for b in range(148)])
for nr in (6, 7):
    sel = (nrows == nr) & (ng == 2)
    if sel.any():
        print(f"2-group CTAs with {nr} rows: {int(sel.sum())}, own work mean {np.nanmean(own[sel]):.2f}")
