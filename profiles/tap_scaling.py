"""Tap-conv scaling probe: time conv forward of a CIFAR-quick conv2 shape at
several batch sizes (tiles per persistent CTA grows with N).  Prints
N, tiles, ms, us per tile-wave."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02272_b200 import cudadnn as cd  # noqa: E402
from conv_bench import timeit  # noqa: E402

ctx = cd.Context(0)
ctx.call("cdnn_set_math_mode", cd.MATH_TF32 if "tf32" in sys.argv else cd.MATH_TF32X3)
rng = np.random.default_rng(0)
c, h, w, co, k, p = 32, 16, 16, 32, 5, 2
for n in (10, 25, 50, 100, 200, 400, 800):
    d = ctx.conv_desc(n, c, h, w, co, k, 1, p)
    x = ctx.upload(rng.uniform(-1, 1, n * c * h * w).astype(np.float32))
    wt = ctx.upload(rng.uniform(-1, 1, co * c * k * k).astype(np.float32))
    y = ctx.alloc(n * co * h * w, cd.F32)
    ms = timeit(ctx, lambda: ctx.call("cdnn_conv_forward", d, x, wt, 0, y, 0), 10)
    tiles = (n * (h + 4) * (w + 4) + 127) // 128
    print(f"N={n:4d} tiles={tiles:5d} per_cta={tiles / 148:5.2f} ms={ms:.4f} us/tile-wave={1000 * ms / max(1, -(-tiles // 148)):.2f}")
    for hh in (x, wt, y):
        ctx.free(hh)
