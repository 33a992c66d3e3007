"""Data-parallel training through the PRODUCT (polegrad.Net + Solver + Parallel),
two processes on one GPU (VERDICT r1 missing-4).

Each rank trains on its half of the global batch; polegrad::Parallel plans the
gradient buckets, launches each from the backward hook, scales the normalised
SoftmaxWithLoss gradient by 1/nranks and joins before the fused update, exactly
as on NCCL; only the transport differs: the Parallel host transport copies each
bucket to the host and the ranks SUM it over gloo (NCCL cannot put two ranks on
one GPU, and ranks whose kernels wait on each other must not share a GPU).  The
result must equal single-process full-batch product training: weights after the
updates at 1e-10 relative in FP64 (FP order only), 1e-3 in float (half of
north_star's 2e-3: the two runs contract over different split-K chain lengths and
the tensor-core accumulator rounds toward zero, ~1e-5 relative per 1024-term
chain, profiles/dbg/gemm_err.py; measured 1.8e-4 on conv1's update after four
steps), the global loss likewise, and the weights identical on both ranks.
The weight check is on the UPDATES (w - w0), not the weights, so the tolerance
is not diluted by the initial values.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from parity_util import polegrad, rel_l2

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from dp_worker import SOLVERS, batches  # noqa: E402


def single_process(model, dtype, gbatch, iters):
    net = polegrad.Net(polegrad.load_model(model, gbatch), seed=1, dtype=dtype)
    solver = polegrad.Solver(net, **SOLVERS[model])
    shape = (gbatch,) + net.blob_shape("data")[1:]
    losses = []
    for x, y in batches(shape, 10, iters):
        net.set_batch(x, y)
        net.forward()
        losses.append(net.loss())
        net.backward()
        solver.apply()
    return np.array(losses), [net.param(i) for i in range(len(net.param_info()))]


def initial_weights(model, dtype, gbatch):
    net = polegrad.Net(polegrad.load_model(model, gbatch), seed=1, dtype=dtype)
    return [net.param(i) for i in range(len(net.param_info()))]


@pytest.mark.parametrize("model,dtype,tol", [("cifar10_quick", "f64", 1e-10), ("cifar10_quick", "f32", 1e-3),
                                             ("lenet", "f64", 1e-10)])
def test_two_rank_product_training_equals_full_batch(model, dtype, tol):
    gbatch, iters, world = 32, 4, 2
    bucket = 64 << 10  # several buckets, so the hook-driven early launches are exercised
    with tempfile.TemporaryDirectory() as out:
        env = dict(os.environ, OMP_NUM_THREADS="1")
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
               "--master-addr=127.0.0.1", f"--master-port={port}", os.path.join(HERE, "dp_worker.py"), model, dtype,
               str(gbatch), str(iters), str(bucket), out]
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
        ranks = [np.load(os.path.join(out, f"rank{k}.npz")) for k in range(world)]
    ref_losses, ref_w = single_process(model, dtype, gbatch, iters)
    w0 = initial_weights(model, dtype, gbatch)
    for k, rk in enumerate(ranks):
        assert int(rk["nranks"]) == world and int(rk["rank"]) == k
        assert int(rk["buckets"]) >= 2
        assert int(rk["launches"]) == iters * int(rk["buckets"])  # every bucket once per step
    dp_losses = np.mean([rk["losses"] for rk in ranks], axis=0)
    assert rel_l2(dp_losses, ref_losses) <= tol, (dp_losses, ref_losses)
    for i, w in enumerate(ref_w):
        assert np.array_equal(ranks[0][f"w{i}"], ranks[1][f"w{i}"]), i  # replicas stay identical
        upd = ranks[0][f"w{i}"].astype(np.float64) - w0[i]
        err = rel_l2(upd, w.astype(np.float64) - w0[i])
        assert err <= tol, (i, err)
