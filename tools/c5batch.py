"""One batched C5 sweep point (64 x 512^2, M=16) for ncu launch lists."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_13049_b200 as fw  # noqa: E402
from paper_2311_13049_b200 import configs  # noqa: E402

ctx = fw.Context(0)
fields = [configs.c5_field(f) for f in range(configs.C5_FIELDS)]
g = fw.Grid(list(zip(fields[0].lo, fields[0].hi)), fields[0].J)
ops = [fw.build_expansion(fw.OrderField(g, f.s), 16, ctx=ctx) for f in fields]
us = [torch.from_numpy(np.ascontiguousarray(f.u)).cuda() for f in fields]
outs = [torch.empty_like(u) for u in us]
for _ in range(3):
    fw.apply_batch_device(ops, [u.data_ptr() for u in us], [o.data_ptr() for o in outs])
ctx.sync()
