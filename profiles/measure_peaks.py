"""Dense TF32 and FP64 tensor-core / DMMA peaks of THIS B200, the roofline
denominators the bench's `roofline.peak` uses for the float (3xTF32 / TF32) and
double paths (MEASURED_PEAKS.json only carries bf16 and HBM).  Same method as
MEASURED_PEAKS.json: torch.matmul 8192^3 (2*N^3 FLOP), best of 10 (burst) and
back to back for 4 s (sustained), CUDA events; TF32 via
torch.backends.cuda.matmul.allow_tf32 (cuBLAS TF32 tensor cores).  bf16 is
re-measured beside them as a cross-check of the box.  Tooling, not product.

    python profiles/measure_peaks.py [out.json]
"""
import json
import sys
import time

import torch


def rate(dtype, n=8192, burst=10, sustain_s=4.0):
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    c = torch.empty(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(burst):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        torch.matmul(a, b, out=c)
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    flop = 2.0 * n ** 3
    # sustained: back to back for sustain_s seconds
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    iters = 0
    s.record()
    while time.time() - t0 < sustain_s:
        for _ in range(8):
            torch.matmul(a, b, out=c)
        iters += 8
        torch.cuda.synchronize() if iters % 64 == 0 else None
    e.record()
    e.synchronize()
    return {"burst_tflops": round(flop / (best / 1e3) / 1e12, 1),
            "sustained_tflops": round(flop * iters / (s.elapsed_time(e) / 1e3) / 1e12, 1)}


def main():
    torch.backends.cuda.matmul.allow_tf32 = True
    torch.backends.cudnn.allow_tf32 = True
    out = {"gpu": torch.cuda.get_device_name(0),
           "how": "torch.matmul 8192^3, 2*N^3 FLOP; burst = best of 10 (CUDA events), "
                  "sustained = back to back for 4 s; TF32 = fp32 inputs with allow_tf32 (cuBLAS TF32)",
           "tf32": rate(torch.float32), "fp64": rate(torch.float64, n=8192, burst=5, sustain_s=3.0),
           "bf16": rate(torch.bfloat16)}
    print(json.dumps(out))
    if len(sys.argv) > 1:
        with open(sys.argv[1], "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
