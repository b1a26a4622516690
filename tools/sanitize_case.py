"""One small case of each kernel family for compute-sanitizer (memcheck / synccheck / racecheck):
the persistent 2D kernel at 512 x 1024 (apply and 2 seismic steps), the multi-pass 3D pipeline at
64 x 32 x 256 (k_rows_r2c, k_lines, k_lines_terms, k_rows_c2r), the full-spectrum path at 40 x 30.
usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py [persistent|multipass|full|all]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_13049_b200 as fw  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
rng = np.random.default_rng(0)
if which in ("persistent", "all"):
    J = (512, 1024)
    g = fw.Grid([(-16.0, 16.0)] * 2, J)
    s = 1.0 + 0.2 * np.sin(np.linspace(0, 6, J[0] * J[1])).reshape(J)
    op = fw.build_expansion(fw.OrderField(g, s), 8)
    assert op.persistent
    out = op.apply(rng.standard_normal(J))
    gamma = np.full(J, 0.02)
    st = fw.SeismicStepper(fw.build_medium(g, gamma, np.ones(J), 1.0, 8), np.exp(-np.linspace(-4, 4, J[0] * J[1]) ** 2).reshape(J),
                           np.zeros(J), 1e-3)
    st.advance(2)
    print("persistent ok", float(np.abs(out).max()), st.n())
if which in ("multipass", "all"):
    J = (64, 32, 256)
    g = fw.Grid([(-4.0, 4.0)] * 3, J)
    s = 1.0 + 0.2 * np.sin(np.linspace(0, 6, int(np.prod(J)))).reshape(J)
    op = fw.build_expansion(fw.OrderField(g, s), 8)
    out = op.apply(rng.standard_normal(J))
    print("multipass ok", float(np.abs(out).max()))
if which in ("full", "all"):
    J = (40, 30)
    g = fw.Grid([(-4.0, 4.0)] * 2, J)
    op = fw.build_expansion(fw.OrderField(g, np.full(J, 1.2) + 0.1 * rng.standard_normal(J) * 0.1), 6)
    out = op.apply(rng.standard_normal(J))
    print("full ok", float(np.abs(out).max()))
os._exit(0)
