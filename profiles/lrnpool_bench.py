"""Device timing of AlexNet's LRN -> MAX pooling pairs through the C-ABI: unfused
(cdnn_lrn_forward + cdnn_pool_forward; cdnn_pool_backward + cdnn_lrn_backward_ex)
against fused (cdnn_lrn_pool_forward / _backward), CUDA events, median of N, with
the achieved algorithmic HBM bandwidth of the fused kernels (bytes: forward reads x
and writes the LRN top, the pooled top and the int32 mask; backward reads x, the
pooled diff and the mask and writes dx).  The tensors exceed the 126 MB L2.

Usage: python profiles/lrnpool_bench.py [--reps 10] [--only norm1] [--fused-only]"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02272_b200 import cudadnn as cd  # noqa: E402

CASES = {"norm1": (256, 96, 55, 55), "norm2": (256, 256, 27, 27)}


def timeit(ctx, fn, reps):
    evs = [(ctx.event(), ctx.event()) for _ in range(reps)]
    fn()
    ctx.sync()
    for a, b in evs:
        ctx.record(a)
        fn()
        ctx.record(b)
    ctx.sync()
    return statistics.median(ctx.elapsed_ms(a, b) for a, b in evs)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--only", default="")
    ap.add_argument("--fused-only", action="store_true")
    args = ap.parse_args()
    ctx = cd.Context(0)
    rng = np.random.default_rng(0)
    size, alpha, beta, k = 5, 1e-4, 0.75, 1.0
    for name, (n, c, h, w) in CASES.items():
        if args.only and args.only != name:
            continue
        d = ctx.pool_desc(n, c, h, w, cd.POOL_MAX, 3, 2)
        _, _, P, Q = ctx.pool_output_shape(d)
        nin, nout = n * c * h * w, n * c * P * Q
        x = ctx.upload(np.maximum(rng.standard_normal(nin), 0).astype(np.float32))
        y, sc, dn, dx = (ctx.alloc(nin, cd.F32) for _ in range(4))
        yp, m, dyp = ctx.alloc(nout, cd.F32), ctx.alloc(nout, cd.I32), ctx.upload(
            rng.standard_normal(nout).astype(np.float32))
        ops = {
            "fused.fwd": (lambda: ctx.call("cdnn_lrn_pool_forward", d, x, y, yp, m, size, alpha, beta, k, 0, 0),
                          4 * (2 * nin + 2 * nout)),
            "fused.bwd": (lambda: ctx.call("cdnn_lrn_pool_backward", d, x, dyp, m, dx, x, size, alpha, beta, k, 0),
                          4 * (2 * nin + 2 * nout)),
        }
        if not args.fused_only:
            ops["unfused.fwd"] = (lambda: (ctx.call("cdnn_lrn_forward", x, y, sc, n, c, h * w, size, alpha, beta, k, 0),
                                           ctx.call("cdnn_pool_forward", d, y, yp, m, 0)), 4 * (4 * nin + 2 * nout))
            ops["unfused.bwd"] = (lambda: (ctx.call("cdnn_pool_backward", d, dyp, m, dn, 0),
                                           ctx.call("cdnn_lrn_backward_ex", x, y, sc, dn, dx, n, c, h * w, size, alpha,
                                                    beta, x, 0)), 4 * (6 * nin + 2 * nout))
        for op, (fn, nbytes) in ops.items():
            ms = timeit(ctx, fn, args.reps)
            print(json.dumps({"op": f"{name}.{op}", "ms": round(ms, 5), "GB/s": round(nbytes / ms / 1e6, 1),
                              "bytes": nbytes}), flush=True)
        for hnd in (x, y, sc, dn, dx, yp, m, dyp):
            ctx.free(hnd)
    ctx.close()


if __name__ == "__main__":
    main()
