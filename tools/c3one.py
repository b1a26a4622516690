"""One C3 (256^3, M=16) apply through the generic multi-pass kernels (for ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_13049_b200 as fw  # noqa: E402
from paper_2311_13049_b200 import configs  # noqa: E402

cfg = configs.c3()
ctx = fw.Context(0)
g = fw.Grid(list(zip(cfg.lo, cfg.hi)), cfg.J)
op = fw.build_expansion(fw.OrderField(g, 1.0 + cfg.gamma), cfg.M, ctx=ctx)
u = torch.from_numpy(np.ascontiguousarray(cfg.phi)).cuda()
o = torch.empty_like(u)
for _ in range(3):
    op.apply_device(u.data_ptr(), o.data_ptr())
ctx.sync()
