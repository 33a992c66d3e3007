"""Per-op device timing of the MAX / AVE pooling kernels of the bench workloads through
the C-ABI (CUDA events on the context stream, median of N launches) with the
achieved algorithmic HBM bandwidth, plus a SHA-1 of every output so two runs
(default kernels vs CDNN_POOL_GENERIC=1) can be compared bit for bit.

Algorithmic bytes: forward reads x once and writes y and (MAX) the int32 mask;
backward (fused ReLU gate) reads dy, (MAX) the mask and the gate, and writes dx.
AlexNet tensors exceed the 126 MB L2; the small CIFAR / LeNet ones are L2-warm.

Usage: python profiles/pool_bench.py [--reps 20]"""
import argparse
import hashlib
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02272_b200 import cudadnn as cd  # noqa: E402

CASES = {
    # name: n, c, h, w, kernel, stride
    "alexnet.pool1": (256, 96, 55, 55, 3, 2),
    "alexnet.pool2": (256, 256, 27, 27, 3, 2),
    "alexnet.pool5": (256, 256, 13, 13, 3, 2),
    "cq.pool1": (100, 32, 32, 32, 3, 2),
    "lenet.pool1": (64, 20, 24, 24, 2, 2),
    "cq.pool2.ave": (100, 32, 16, 16, 3, 2),
    "cq.pool3.ave": (100, 64, 8, 8, 3, 2),
}


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
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    ctx = cd.Context(0)
    rng = np.random.default_rng(0)
    variant = "generic" if os.environ.get("CDNN_POOL_GENERIC") == "1" else "default"
    for name, (n, c, h, w, k, s) in CASES.items():
        ave = name.endswith(".ave")
        d = ctx.pool_desc(n, c, h, w, cd.POOL_AVE if ave else cd.POOL_MAX, k, s)
        _, _, P, Q = ctx.pool_output_shape(d)
        nin, nout = n * c * h * w, n * c * P * Q
        x = ctx.upload(rng.uniform(-1, 1, nin).astype(np.float32))
        y = ctx.alloc(nout, cd.F32)
        m = ctx.alloc(nout, cd.I32)
        dy = ctx.upload(rng.uniform(-1, 1, nout).astype(np.float32))
        dx = ctx.alloc(nin, cd.F32)
        ops = {
            "fwd": (lambda: ctx.call("cdnn_pool_forward", d, x, y, 0 if ave else m, 0), 4 * (nin + (1 if ave else 2) * nout)),
            "bwd_gate": (lambda: ctx.call("cdnn_pool_backward_ex", d, dy, 0 if ave else m, dx, x, 0),
                         4 * ((1 if ave else 2) * nout + 2 * nin)),
        }
        for op, (fn, nbytes) in ops.items():
            ms = timeit(ctx, fn, args.reps)
            outs = ((y,) if ave else (y, m)) if op == "fwd" else (dx,)
            sha = hashlib.sha1(b"".join(ctx.read(o).tobytes() for o in outs)).hexdigest()[:16]
            print(json.dumps({"op": f"{name}.{op}", "variant": variant, "us": round(ms * 1e3, 2),
                              "gbps": round(nbytes / ms / 1e6, 1), "mb": round(nbytes / 1e6, 2), "sha1": sha}),
                  flush=True)
        for hnd in (x, y, m, dy, dx):
            ctx.free(hnd)
        ctx.call("cdnn_desc_free", d)
    ctx.close()


if __name__ == "__main__":
    main()
