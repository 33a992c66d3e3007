"""Per-op device timing of the convolution / InnerProduct contractions of the
bench workloads through the C-ABI (CUDA events on the context stream, median
of N launches, L2-warm).  Prints one JSON line per op.

Usage: python profiles/conv_bench.py [--math tf32x3|tf32] [--reps 20]"""
import argparse
import ctypes as C
import json
import os
import statistics
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1810_02272_b200 import cudadnn as cd  # noqa: E402

CASES = {
    # name: n, c, h, w, co, k, stride, pad[, group]
    "cq.conv1": (100, 3, 32, 32, 32, 5, 1, 2),
    "cq.conv2": (100, 32, 16, 16, 32, 5, 1, 2),
    "cq.conv3": (100, 32, 8, 8, 64, 5, 1, 2),
    "lenet.conv1": (64, 1, 28, 28, 20, 5, 1, 0),
    "lenet.conv2": (64, 20, 12, 12, 50, 5, 1, 0),
    "rn.stage1": (128, 16, 32, 32, 16, 3, 1, 1),
    "rn.stage3": (128, 64, 8, 8, 64, 3, 1, 1),
    "alexnet.conv1": (256, 3, 227, 227, 96, 11, 4, 0),
    "alexnet.conv2": (256, 96, 27, 27, 256, 5, 1, 2, 2),
    "alexnet.conv3": (256, 256, 13, 13, 384, 3, 1, 1),
    "alexnet.conv4": (256, 384, 13, 13, 384, 3, 1, 1, 2),
    "alexnet.conv5": (256, 384, 13, 13, 256, 3, 1, 1, 2),
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
    ap.add_argument("--math", default="tf32x3")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--ops", default="", help="comma list of ops to time (fwd,dgrad,wgrad,dgrad_gate,bwd)")
    args = ap.parse_args()
    ctx = cd.Context(0)
    ctx.call("cdnn_set_math_mode", cd.MATH_TF32X3 if args.math == "tf32x3" else cd.MATH_TF32)
    rng = np.random.default_rng(0)
    for name, case in CASES.items():
        n, c, h, w, co, k, s, p = case[:8]
        g = case[8] if len(case) > 8 else 1
        if args.only and args.only not in name:
            continue
        d = ctx.conv_desc(n, c, h, w, co, k, s, p, 1, g)
        _, _, P, Q = ctx.conv_output_shape(d)
        x = ctx.upload(rng.uniform(-1, 1, n * c * h * w).astype(np.float32))
        wt = ctx.upload(rng.uniform(-1, 1, co * c // g * k * k).astype(np.float32))
        b = ctx.upload(np.zeros(co, np.float32))
        y = ctx.alloc(n * co * P * Q, cd.F32)
        dy = ctx.upload(rng.uniform(-1, 1, n * co * P * Q).astype(np.float32))
        dx = ctx.alloc(n * c * h * w, cd.F32)
        dw = ctx.alloc(co * c // g * k * k, cd.F32)
        db = ctx.alloc(co, cd.F32)
        flops = 2.0 * n * P * Q * co * c // g * k * k
        ops = {
            "fwd": lambda: ctx.call("cdnn_conv_forward", d, x, wt, b, y, 0),
            "dgrad": lambda: ctx.call("cdnn_conv_backward_data", d, wt, dy, dx, 0),
            "wgrad": lambda: ctx.call("cdnn_conv_backward_filter", d, x, dy, dw, 0, 0),
            # backward-data with the fused ReLU gate (gate = the layer's own input here)
            "dgrad_gate": lambda: ctx.call("cdnn_conv_backward_data_ex", d, wt, dy, dx, x, 0),
        }
        for op, fn in ops.items():
            if args.ops and op not in args.ops.split(","):
                continue
            ms = timeit(ctx, fn, args.reps)
            print(json.dumps({"op": f"{name}.{op}", "math": args.math, "ms": round(ms, 5),
                              "tflops": round(flops / ms / 1e9, 3), "gflop": round(flops / 1e9, 4)}), flush=True)
        for hnd in (x, wt, b, y, dy, dx, dw, db):
            ctx.free(hnd)
    # InnerProduct layers (forward, backward = dW + db + dX) of AlexNet / CIFAR-quick
    IP = {"alexnet.fc6": (256, 9216, 4096), "alexnet.fc7": (256, 4096, 4096), "alexnet.fc8": (256, 4096, 1000),
          "cq.ip1": (100, 1024, 64)}
    for name, (rows, k, o) in IP.items():
        if args.only and args.only not in name:
            continue
        x = ctx.upload(rng.uniform(-1, 1, rows * k).astype(np.float32))
        wt = ctx.upload(rng.uniform(-1, 1, o * k).astype(np.float32))
        b = ctx.upload(np.zeros(o, np.float32))
        y = ctx.alloc(rows * o, cd.F32)
        dy = ctx.upload(rng.uniform(-1, 1, rows * o).astype(np.float32))
        dx = ctx.alloc(rows * k, cd.F32)
        dw = ctx.alloc(o * k, cd.F32)
        db = ctx.alloc(o, cd.F32)
        flops = 2.0 * rows * k * o
        ops = {
            "fwd": (lambda: ctx.call("cdnn_ip_forward", x, wt, b, y, rows, k, o, 0, 0), flops),
            "bwd": (lambda: ctx.call("cdnn_ip_backward", x, wt, dy, dw, db, dx, rows, k, o, 0), 2 * flops),
        }
        for op, (fn, fl) in ops.items():
            if args.ops and op not in args.ops.split(","):
                continue
            ms = timeit(ctx, fn, args.reps)
            print(json.dumps({"op": f"{name}.{op}", "math": args.math, "ms": round(ms, 5),
                              "tflops": round(fl / ms / 1e9, 3), "gflop": round(fl / 1e9, 4)}), flush=True)
        for hnd in (x, wt, b, y, dy, dx, dw, db):
            ctx.free(hnd)
    ctx.close()


if __name__ == "__main__":
    main()
