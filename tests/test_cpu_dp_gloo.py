"""Data-parallel protocol on the CPU, world_size 2 over gloo (127.0.0.1).

Runs exactly what polegrad::Parallel does on NCCL, with the oracle as the
per-rank compute: each rank takes its slice of the global batch, scales the
SoftmaxWithLoss gradient by 1/nranks (Net::set_loss_scale), all-reduces the
flat gradient arena SUM in the buckets planned by polegrad::plan_buckets
(reverse parameter order), and applies the same momentum-SGD update.  The
result must equal one process training on the whole batch, and the weights
must stay identical on both ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from parity_util import pyoracle, polegrad

pytestmark = pytest.mark.skipif(not pyoracle.available("f64"), reason="oracle/_ref not built")

GLOBAL = 8
WORLD = 2


def model(batch):
    return polegrad.load_model("cifar10_quick").replace("batch_size: 100", f"batch_size: {batch}")


def batches(steps=3):
    rng = np.random.default_rng(2)
    return [(rng.uniform(-1, 1, (GLOBAL, 3, 32, 32)), np.floor(rng.uniform(0, 1, GLOBAL) * 10)) for _ in range(steps)]


def arena_layout(shapes):
    counts = [int(np.prod(s)) for s in shapes]
    offs, o = [], 0
    for c in counts:
        offs.append(o)
        o += (c + 3) // 4 * 4  # Net::pack_params 16-byte alignment
    return offs, counts, o


def _worker(rank, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    local = GLOBAL // WORLD
    net = pyoracle.OracleNet(model(local), 1, "f64")
    solver = pyoracle.OracleSolver(net, "sgd", 0.001, momentum=0.9, weight_decay=0.004)
    shapes = [s for _, s in net.param_info()]
    offs, counts, total = arena_layout(shapes)
    bucket_of, nb = polegrad.plan_buckets(offs, counts, total, 4096)
    for x, y in batches():
        sl = slice(rank * local, (rank + 1) * local)
        net.set_batch(x[sl], y[sl])
        net.forward()
        net.backward()
        arena = np.zeros(total)
        for i, c in enumerate(counts):
            arena[offs[i]:offs[i] + c] = net.param(i, True).ravel() / WORLD  # loss scale 1/nranks
        # buckets in the order backward completes them: bucket 0 holds the last parameters
        for b in range(nb):
            members = [i for i in range(len(counts)) if bucket_of[i] == b]
            lo, hi = min(offs[i] for i in members), max(offs[i] + counts[i] for i in members)
            t = torch.from_numpy(arena[lo:hi].copy())
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            arena[lo:hi] = t.numpy()
        for i, c in enumerate(counts):
            net.set_param(i, arena[offs[i]:offs[i] + c].reshape(shapes[i]), diff=True)
        solver.apply()
    w = np.concatenate([net.param(i).ravel() for i in range(len(counts))])
    out[rank] = w
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_sum_allreduce_equals_single_process():
    mgr = mp.get_context("spawn").Manager()
    out = mgr.dict()
    port = _free_port()
    mp.start_processes(_worker, args=(port, out), nprocs=WORLD, start_method="spawn", join=True)
    # single process, whole batch
    net = pyoracle.OracleNet(model(GLOBAL), 1, "f64")
    solver = pyoracle.OracleSolver(net, "sgd", 0.001, momentum=0.9, weight_decay=0.004)
    for x, y in batches():
        net.set_batch(x, y)
        net.forward()
        net.backward()
        solver.apply()
    ref = np.concatenate([net.param(i).ravel() for i in range(len(net.param_info()))])
    assert np.array_equal(out[0], out[1]), "weights must stay identical across ranks"
    err = np.linalg.norm(out[0] - ref) / np.linalg.norm(ref)
    assert err < 1e-12, err
