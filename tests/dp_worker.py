"""One rank of the product-level data-parallel check (tests/test_gpu_dp_product.py),
launched by torch.distributed.run: polegrad.Net + Solver + Parallel on this rank's
slice of the global batch, the gradient buckets combined across ranks over gloo by
the Parallel host transport.  Writes its losses, final weights and the Parallel
info to <out>/rank<r>.npz.

    python -m torch.distributed.run --nproc-per-node 2 ... tests/dp_worker.py
        <model> <dtype> <global_batch> <iters> <bucket_bytes> <out_dir>
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from paper_1810_02272_b200 import polegrad  # noqa: E402

SOLVERS = {
    "cifar10_quick": dict(method="sgd", lr=0.001, momentum=0.9, weight_decay=4e-3),
    "lenet": dict(method="sgd", lr=0.01, momentum=0.9, weight_decay=5e-4),
}


def batches(shape, classes, iters, seed=2):
    rng = np.random.default_rng(seed)
    return [(rng.uniform(-1.0, 1.0, shape), np.floor(rng.uniform(0.0, 1.0, shape[0]) * classes))
            for _ in range(iters)]


def main():
    model, dtype, gbatch, iters, bucket, out = sys.argv[1:7]
    gbatch, iters, bucket = int(gbatch), int(iters), int(bucket)
    dist.init_process_group("gloo", init_method="env://")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = gbatch // world
    text = polegrad.load_model(model, local)
    net = polegrad.Net(text, seed=1 + rank, dtype=dtype)  # rank 0's weights arrive by broadcast
    solver = polegrad.Solver(net, **SOLVERS[model])

    def transport(op, arr, offset):
        t = torch.from_numpy(arr)
        if op == 0:
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
        else:
            dist.broadcast(t, src=0)

    par = polegrad.Parallel.host(net, world, rank, transport, bucket_bytes=bucket)
    par.broadcast()
    solver.set_parallel(par)
    shape = (gbatch,) + net.blob_shape("data")[1:]
    losses = []
    for x, y in batches(shape, 10, iters):
        net.set_batch(x[rank * local:(rank + 1) * local], y[rank * local:(rank + 1) * local])
        net.forward()
        losses.append(net.loss())
        net.backward()
        solver.apply()
    info = par.info()
    solver.set_parallel(None)
    weights = [net.param(i) for i in range(len(net.param_info()))]
    np.savez(os.path.join(out, f"rank{rank}.npz"), losses=np.array(losses), nranks=info["nranks"],
             rank=info["rank"], buckets=info["buckets"], launches=info["launches"],
             **{f"w{i}": w for i, w in enumerate(weights)})
    par.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
