"""HBM bandwidth a plain torch elementwise kernel reaches at the read:write mixes of the
pooling kernels (forward reads 2.1x what it writes, backward with gate ~1.5:1), next to
the 1:1 copy of MEASURED_PEAKS.json.  CUDA events, best of 20, tensors >> L2."""
import json
import torch

n = 256 * 1024 * 1024 // 4  # 256 MiB fp32 per tensor
dev = "cuda"
a, b, c, d = (torch.rand(n, device=dev) for _ in range(4))
o = torch.empty(n, device=dev)
o2 = torch.empty(n, device=dev)


def best(fn, nbytes):
    ts = []
    for _ in range(22):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); fn(); e.record(); torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    t = min(ts[2:])
    return round(nbytes / (t * 1e-3) / 1e9, 1)


res = {
    "copy 1:1": best(lambda: o.copy_(a), 2 * 4 * n),
    "add 2:1": best(lambda: torch.add(a, b, out=o), 3 * 4 * n),
    "addcmul 3:1": best(lambda: torch.addcmul(a, b, c, out=o), 4 * 4 * n),
    "read-only sum": best(lambda: a.sum(), 4 * n),
}
print(json.dumps({"GB/s": res}))
