"""3xTF32 GEMM error vs K, vs M, and with tf32-exact inputs (isolates accumulation)."""
import sys, numpy as np
sys.path.insert(0, '.')
from paper_1810_02272_b200 import cudadnn as cd
ctx = cd.Context(0)
ctx.call("cdnn_set_math_mode", cd.MATH_TF32X3)
def rel(a, b): return float(np.linalg.norm(a - b) / np.linalg.norm(b))
def tf32(x):
    u = x.astype(np.float32).view(np.uint32) & np.uint32(0xFFFFE000)
    return u.view(np.float32)
def run(m, n, k, exact=False, pos=False, ta=0):
    rng = np.random.default_rng(5)
    lo = 0 if pos else -1
    A = rng.uniform(lo, 1, (m, k)).astype(np.float32); B = rng.uniform(lo, 1, (k, n)).astype(np.float32)
    if exact: A, B = tf32(A), tf32(B)
    Ah = np.ascontiguousarray(A.T) if ta else A
    ha, hb, hc = ctx.upload(Ah), ctx.upload(B), ctx.upload(np.zeros((m, n), np.float32))
    ctx.call("cdnn_gemm", ta, 0, m, n, k, 1.0, ha, hb, 0.0, hc, 0)
    got = ctx.read(hc).reshape(m, n); want = A.astype(np.float64) @ B.astype(np.float64)
    for h in (ha, hb, hc): ctx.free(h)
    return rel(got, want), rel((A @ B), want)
for k in (512, 1024, 2048, 4096, 8192):
    print("K", k, "rand", run(1024, 256, k), "tf32-exact", run(1024, 256, k, exact=True), "positive", run(1024, 256, k, pos=True), flush=True)
for m in (1024, 4096, 9216):
    print("M", m, "K4096", run(m, 256, 4096), "ta", run(m, 256, 4096, ta=1), flush=True)
