"""Time the feed ring's in-graph staged-batch copy (cdnn_copy_range: cudaMemcpyAsync D2D)
against cdnn_copy (the library's copy kernel) for AlexNet's 256x3x227x227 batch."""
import json, os, sys, statistics
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1810_02272_b200 import cudadnn as cd
ctx = cd.Context(0)
n = 256 * 3 * 227 * 227
a = ctx.upload(np.ones(n, np.float32))
b = ctx.alloc(n, cd.F32)
def t(fn, reps=20):
    evs = [(ctx.event(), ctx.event()) for _ in range(reps)]
    fn(); ctx.sync()
    for s, e in evs:
        ctx.record(s); fn(); ctx.record(e)
    ctx.sync()
    return statistics.median(ctx.elapsed_ms(s, e) for s, e in evs)
r = {"memcpy_d2d_us": 1e3 * t(lambda: ctx.call("cdnn_copy_range", a, 0, b, 0, n, 0)),
     "copy_kernel_us": 1e3 * t(lambda: ctx.call("cdnn_copy", a, b, n, 0)), "bytes": 8 * n}
print(json.dumps(r))
