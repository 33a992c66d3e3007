"""Which InnerProduct-backward GEMM fails at AlexNet fc shapes (dX only / dW only)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1810_02272_b200 import cudadnn as cd
rows, k, o = [int(v) for v in sys.argv[1:4]]
which = sys.argv[4]
ctx = cd.Context(0)
rng = np.random.default_rng(0)
x = ctx.upload(rng.uniform(-1, 1, rows * k).astype(np.float32))
w = ctx.upload(rng.uniform(-1, 1, o * k).astype(np.float32))
dy = ctx.upload(rng.uniform(-1, 1, rows * o).astype(np.float32))
dx = ctx.alloc(rows * k, cd.F32)
dw = ctx.upload(np.zeros(o * k, np.float32))
db = ctx.upload(np.zeros(o, np.float32))
if which == "dx":
    ctx.call("cdnn_ip_backward", x, w, dy, 0, 0, dx, rows, k, o, 0)
elif which == "both":
    for _ in range(int(os.environ.get("REPS", "1"))):
        ctx.call("cdnn_ip_backward", x, w, dy, dw, db, dx, rows, k, o, 0)
elif which == "dw":
    ctx.call("cdnn_ip_backward", x, w, dy, dw, db, 0, rows, k, o, 0)
else:
    ctx.call("cdnn_ip_forward", x, w, db, dx if False else ctx.alloc(rows * o, cd.F32), rows, k, o, 0, 0)
ctx.sync()
print(which, rows, k, o, "ok")
