"""debug: conv fwd/dgrad/wgrad rel errors vs torch fp64 for a shape list (prints one line each)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1810_02272_b200 import cudadnn as cd
ctx = cd.Context(0)
ctx.call("cdnn_set_math_mode", int(os.environ.get("MATH", "1")))
rng = np.random.default_rng(0)
def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
for shape in [(64,1,28,28,20,5,1,0),(64,20,12,12,50,5,1,0),(100,3,32,32,32,5,1,2),(100,32,16,16,32,5,1,2),(100,32,8,8,64,5,1,2),(3,5,13,20,7,3,1,1)]:
    n, c, h, w, co, k, s, p = shape
    x = rng.uniform(-1, 1, (n, c, h, w)); wt = rng.uniform(-1, 1, (co, c, k, k))
    d = ctx.conv_desc(n, c, h, w, co, k, s, p); shp = ctx.conv_output_shape(d)
    xt = torch.from_numpy(x).requires_grad_(); wtt = torch.from_numpy(wt).requires_grad_()
    y = torch.nn.functional.conv2d(xt, wtt, stride=s, padding=p); dy = rng.uniform(-1, 1, tuple(y.shape)); y.backward(torch.from_numpy(dy))
    hx, hw, hy = ctx.upload(x.astype(np.float32)), ctx.upload(wt.astype(np.float32)), ctx.alloc(int(np.prod(shp)), cd.F32)
    hdy, hdx = ctx.upload(dy.astype(np.float32)), ctx.alloc(x.size, cd.F32)
    ctx.call("cdnn_conv_forward", d, hx, hw, 0, hy, 0)
    ctx.call("cdnn_conv_backward_data", d, hw, hdy, hdx, 0)
    gy, gdx = ctx.read(hy).reshape(shp), ctx.read(hdx).reshape(x.shape)
    ey = np.abs(gy - y.detach().numpy()); edx = np.abs(gdx - xt.grad.numpy())
    print(shape, "fwd", rel(gy, y.detach().numpy()), "worst@", np.unravel_index(ey.argmax(), ey.shape),
          "dgrad", rel(gdx, xt.grad.numpy()), "worst@", np.unravel_index(edx.argmax(), edx.shape))
