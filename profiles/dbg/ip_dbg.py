import sys, numpy as np
sys.path.insert(0, '.')
from paper_1810_02272_b200 import cudadnn as cd
ctx = cd.Context(0)
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
for math in ("tf32x3", "tf32"):
    ctx.call("cdnn_set_math_mode", cd.MATH_TF32X3 if math == "tf32x3" else cd.MATH_TF32)
    for rows, k, o in [(256, 9216, 4096), (256, 4096, 4096), (96, 6000, 1100), (256, 4096, 1000)]:
        rng = np.random.default_rng(1)
        X = rng.uniform(-1, 1, (rows, k)).astype(np.float32)
        W = rng.uniform(-1, 1, (o, k)).astype(np.float32)
        dY = rng.uniform(-1, 1, (rows, o)).astype(np.float32)
        hx, hw, hdy = ctx.upload(X), ctx.upload(W), ctx.upload(dY)
        hdw, hdb, hdx = ctx.upload(np.zeros((o, k), np.float32)), ctx.alloc(o, cd.F32), ctx.alloc(rows * k, cd.F32)
        ctx.call("cdnn_ip_backward", hx, hw, hdy, hdw, hdb, hdx, rows, k, o, 0)
        dx = ctx.read(hdx).reshape(rows, k); dw = ctx.read(hdw).reshape(o, k)
        rdx = dY.astype(np.float64) @ W.astype(np.float64); rdw = dY.T.astype(np.float64) @ X.astype(np.float64)
        bad = np.argwhere(np.abs(dx - rdx) > 1e-3 * np.abs(rdx).max())
        print(math, rows, k, o, "dx", rel(dx, rdx), "dw", rel(dw, rdw), "bad dx", len(bad), bad[:3].tolist(),
              "bad rows", np.unique(bad[:, 0])[:10].tolist() if len(bad) else [], "bad cols", np.unique(bad[:, 1] // 128)[:10].tolist() if len(bad) else [], flush=True)
        for h in (hx, hw, hdy, hdw, hdb, hdx): ctx.free(h)
