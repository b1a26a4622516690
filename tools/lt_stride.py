"""All-terms axis-0 inverse (k_lines_terms via fw_stage_c2c, w fused, 17 terms) on slabs of
different shapes: effective HBM bandwidth against the axis-0 stride J1 (J2/2+1) complex.
usage: python tools/lt_stride.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_13049_b200 as fw  # noqa: E402
from paper_2311_13049_b200 import slab  # noqa: E402

ctx = fw.Context(0)
st = slab.DeviceStages(ctx)
nt = 17
for shape in [(512, 8, 512), (512, 32, 512), (512, 64, 512), (512, 128, 512), (512, 256, 512), (512, 512, 512),
              (256, 256, 256), (1024, 64, 512)]:
    h = shape[2] // 2 + 1
    nh = shape[0] * shape[1] * h
    u = torch.randn(shape[0], shape[1], h, dtype=torch.complex128, device="cuda")
    w = torch.rand(nt, nh, dtype=torch.float64, device="cuda")
    for _ in range(2):
        out = st.c2c(u, shape, 0, +1, w=w, nterms=nt, w_ts=1)
    ctx.sync()
    s = torch.cuda.ExternalStream(ctx.stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record(s)
    for _ in range(reps):
        out = st.c2c(u, shape, 0, +1, w=w, nterms=nt, w_ts=1)
    e1.record(s)
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    by = nh * 16 + nt * nh * 8 + nt * nh * 16
    print(f"{shape}: stride {shape[1] * h * 16 / 1024:8.0f} KiB  {ms:8.3f} ms  {by / ms / 1e6:7.0f} GB/s", flush=True)
    del u, w, out
    torch.cuda.empty_cache()
