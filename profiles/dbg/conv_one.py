"""debug: one conv forward through the C-ABI; prints rel error vs torch."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1810_02272_b200 import cudadnn as cd
n, c, h, w, co, k, s, p = [int(v) for v in sys.argv[1:9]]
ctx = cd.Context(0)
ctx.call("cdnn_set_math_mode", int(sys.argv[9]) if len(sys.argv) > 9 else 1)
rng = np.random.default_rng(0)
x = rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32); wt = rng.uniform(-1, 1, (co, c, k, k)).astype(np.float32)
d = ctx.conv_desc(n, c, h, w, co, k, s, p)
shp = ctx.conv_output_shape(d)
hx, hw, hy = ctx.upload(x), ctx.upload(wt), ctx.alloc(int(np.prod(shp)), cd.F32)
ctx.call("cdnn_conv_forward", d, hx, hw, 0, hy, 0)
ref = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(wt).double(), stride=s, padding=p).numpy()
got = ctx.read(hy).reshape(shp)
print("dbg", os.environ.get("CDNN_CONV_TMA_DBG"), "rel err", np.linalg.norm(got - ref) / np.linalg.norm(ref))
