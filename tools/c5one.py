import numpy as np, torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_2311_13049_b200 as fw
from paper_2311_13049_b200 import configs
ctx = fw.Context(0)
f = configs.c5_field(0)
g = fw.Grid(list(zip(f.lo, f.hi)), f.J)
op = fw.build_expansion(fw.OrderField(g, f.s), 16, ctx=ctx)
u = torch.from_numpy(np.ascontiguousarray(f.u)).cuda(); o = torch.empty_like(u)
for _ in range(5): op.apply_device(u.data_ptr(), o.data_ptr())
ctx.sync()
