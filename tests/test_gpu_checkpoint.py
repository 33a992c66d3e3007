"""Checkpoint / resume: MCWT weights + MCSS solver state
taken mid-run restore into a fresh Net and Solver, and the resumed run is bit
identical to the uninterrupted one (same kernels, deterministic reductions)."""
import ctypes as C

import numpy as np
import pytest

from parity_util import CONFIGS, data_shape, polegrad, synthetic_batches
from paper_1810_02272_b200 import cudadnn

pytestmark = pytest.mark.gpu


def step(net, solver, x, y, labelled):
    if labelled:
        net.set_batch(x, y)
    else:
        net.set_batch(x)
    net.forward()
    if labelled:
        net.backward()
    else:
        net.set_blob("logits", np.ones(net.blob_shape("logits")), diff=True)
        net.backward_from("logits")
    solver.apply()


@pytest.mark.parametrize("config,dtype", [("cifar10_quick", "f32"), ("pg_mlp", "f64"), ("resnet20", "f32")])
def test_resume_is_bit_identical(config, dtype):
    model, skw, classes, batch = CONFIGS[config]
    text = polegrad.load_model(model, batch)
    shape, labelled = data_shape(text)
    batches = synthetic_batches(shape, classes, 6, seed=5)
    a = polegrad.Net(text, 1, dtype)
    sa = polegrad.Solver(a, **skw)
    for x, y in batches[:3]:
        step(a, sa, x, y, labelled)
    weights, state = a.snapshot(), sa.snapshot()
    assert sa.iterations == 3
    for x, y in batches[3:]:
        step(a, sa, x, y, labelled)
    b = polegrad.Net(text, 99, dtype)  # different init, overwritten by the checkpoint
    sb = polegrad.Solver(b, **skw)
    b.restore(weights)
    sb.restore(state)
    for x, y in batches[3:]:
        step(b, sb, x, y, labelled)
    assert sb.iterations == 6
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i)), a.param_info()[i]
    assert sa.snapshot() == sb.snapshot()


def test_restore_rejects_other_rule():
    text = polegrad.load_model("pg_mlp")
    net = polegrad.Net(text, 1, "f32")
    s = polegrad.Solver(net, method="rmsprop", lr=1e-3)
    s.apply()
    blob = s.snapshot()
    other = polegrad.Solver(net, method="sgd", lr=1e-3, momentum=0.9)
    with pytest.raises(Exception, match="different update rule"):
        other.restore(blob)


@pytest.mark.parametrize("pinned", [False, True])
@pytest.mark.parametrize("depth", [1, 2, 3])
def test_feed_ring_matches_eager_steps(depth, pinned):
    """The pinned feed ring trains exactly like eager steps, with
    host batches copied into its slots (push) or enqueued from the caller's pinned
    buffers (push_pinned, zero-copy)."""
    text = polegrad.load_model("cifar10_quick")
    batches = synthetic_batches((100, 3, 32, 32), 10, 6, seed=8)
    kw = CONFIGS["cifar10_quick"][1]
    a = polegrad.Net(text, 1, "f32")
    sa = polegrad.Solver(a, **kw)
    b = polegrad.Net(text, 1, "f32")
    sb = polegrad.Solver(b, **kw)
    eager = []
    for x, y in batches:
        a.set_batch(x, y)
        a.forward()
        eager.append(a.loss())
        a.backward()
        sa.apply()
    ring = polegrad.FeedRing(b, sb, depth)
    got, inflight, keep = [], 0, []
    for x, y in batches:
        if inflight == depth:
            got.append(ring.pop_loss())
            inflight -= 1
        if pinned:
            px, py = cudadnn.PinnedBuffer(x.shape), cudadnn.PinnedBuffer(y.shape)
            px.array[...] = x
            py.array[...] = y
            keep.append((px, py))  # unchanged until the step's loss is popped
            ring.push_pinned(px, py)
        else:
            ring.push(x, y)
        inflight += 1
    while inflight:
        got.append(ring.pop_loss())
        inflight -= 1
    assert [np.float32(v) for v in got] == [np.float32(v) for v in eager]
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i))
    with pytest.raises(Exception, match="no step in flight"):
        ring.pop_loss()
    ring.close()


def test_feed_ring_rejects_overfill():
    text = polegrad.load_model("cifar10_quick")
    net = polegrad.Net(text, 1, "f32")
    s = polegrad.Solver(net, method="sgd", lr=1e-3)
    ring = polegrad.FeedRing(net, s, 1)
    (x, y), = synthetic_batches((100, 3, 32, 32), 10, 1)
    ring.push(x, y)
    with pytest.raises(Exception, match="full"):
        ring.push(x, y)
    ring.pop_loss()
    with pytest.raises(Exception, match="wrong number"):
        ring.push(x[:50], y)


@pytest.mark.parametrize("method,use_boost", [("uniform", False), ("label_balanced", True)])
def test_feed_ring_push_sampled_matches_eager(tmp_path, method, use_boost):
    """imagedb -> pinned slot gather: push_sampled trains
    exactly like eager steps on the batches the same Rng seed samples."""
    rs = np.random.RandomState(4)
    entries = [(int(k * 13 + 5), int(rs.randint(0, 10)), float(1 + rs.randint(0, 3)),
                rs.uniform(-1, 1, (3, 32, 32)).astype(np.float32)) for k in range(260)]
    db = polegrad.ImageDB(polegrad.write_imagedb(str(tmp_path), entries))
    by_id = {e[0]: e for e in entries}
    text = polegrad.load_model("cifar10_quick")
    kw = CONFIGS["cifar10_quick"][1]
    steps = 5
    ids = db.sample(polegrad.Rng(77), 100 * steps, method, use_boost).reshape(steps, 100)
    a = polegrad.Net(text, 1, "f32")
    sa = polegrad.Solver(a, **kw)
    eager = []
    for row in ids:
        x = np.stack([by_id[i][3] for i in row])
        y = np.array([by_id[i][1] for i in row], dtype=np.float32)
        a.set_batch(x, y)
        a.forward()
        eager.append(a.loss())
        a.backward()
        sa.apply()
    b = polegrad.Net(text, 1, "f32")
    sb = polegrad.Solver(b, **kw)
    ring = polegrad.FeedRing(b, sb, 2)
    rng = polegrad.Rng(77)
    got = []
    for k in range(steps):
        if k >= 2:
            got.append(ring.pop_loss())
        ring.push_sampled(db, rng, method, use_boost)
    got += [ring.pop_loss(), ring.pop_loss()]
    assert [np.float32(v) for v in got] == [np.float32(v) for v in eager]
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i))
    ring.close()


def test_feed_ring_push_sampled_rejects_wrong_tensor(tmp_path):
    db = polegrad.ImageDB(polegrad.write_imagedb(str(tmp_path), [(1, 0, 1.0, np.zeros((1, 2, 2)))]))
    net = polegrad.Net(polegrad.load_model("cifar10_quick"), 1, "f32")
    ring = polegrad.FeedRing(net, polegrad.Solver(net, method="sgd", lr=1e-3), 1)
    with pytest.raises(Exception, match="sampled entry 1 has 4 values"):
        ring.push_sampled(db, polegrad.Rng(1))


def test_parallel_one_rank_nccl_matches_single_process():
    """polegrad::Parallel end to end on a real NCCL communicator (1 rank on this
    1-GPU box): weight broadcast, bucketed all-reduce on the comm stream hooked
    into the two-stream backward, join before the update.  A 1-rank sum is the
    identity, so training is bit-identical to the plain single-process run."""
    cd = polegrad.cudadnn
    ok = C.c_int()
    cd.load().cdnn_nccl_available(C.byref(ok))
    if not ok.value:
        pytest.skip("NCCL not loadable")
    text = polegrad.load_model("cifar10_quick")
    kw = CONFIGS["cifar10_quick"][1]
    batches = synthetic_batches((100, 3, 32, 32), 10, 4, seed=9)
    a = polegrad.Net(text, 1, "f32")
    sa = polegrad.Solver(a, **kw)
    b = polegrad.Net(text, 1, "f32")
    sb = polegrad.Solver(b, **kw)
    par = polegrad.Parallel(b, 1, 0, polegrad.Parallel.unique_id(), bucket_bytes=64 << 10)
    sb.set_parallel(par)
    par.broadcast()
    for x, y in batches:
        for n, s in ((a, sa), (b, sb)):
            n.set_batch(x, y)
            n.forward()
            n.backward()
            s.apply()
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i)), a.param_info()[i]


def _nccl_or_skip():
    ok = C.c_int()
    polegrad.cudadnn.load().cdnn_nccl_available(C.byref(ok))
    if not ok.value:
        pytest.skip("NCCL not loadable")


def test_feed_ring_with_parallel_captures_every_bucket():
    """FeedRing + Parallel: the ring's warm-up step launches no all-reduce
    (the backward hook is detached), each captured slot contains one all-reduce per
    bucket, and ring training equals eager data-parallel training bit for bit."""
    _nccl_or_skip()
    text = polegrad.load_model("cifar10_quick")
    kw = CONFIGS["cifar10_quick"][1]
    batches = synthetic_batches((100, 3, 32, 32), 10, 5, seed=12)
    a = polegrad.Net(text, 1, "f32")
    sa = polegrad.Solver(a, **kw)
    pa = polegrad.Parallel(a, 1, 0, polegrad.Parallel.unique_id(), bucket_bytes=64 << 10)
    sa.set_parallel(pa)
    b = polegrad.Net(text, 1, "f32")
    sb = polegrad.Solver(b, **kw)
    pb = polegrad.Parallel(b, 1, 0, polegrad.Parallel.unique_id(), bucket_bytes=64 << 10)
    sb.set_parallel(pb)
    nb = pb.info()["buckets"]
    assert nb >= 2
    ring = polegrad.FeedRing(b, sb, 2)
    assert pb.info()["launches"] == 2 * nb  # one per bucket in each captured slot, none from the warm-up
    eager = []
    for x, y in batches:
        a.set_batch(x, y)
        a.forward()
        eager.append(a.loss())
        a.backward()
        sa.apply()
    got, inflight = [], 0
    for x, y in batches:
        if inflight == 2:
            got.append(ring.pop_loss())
            inflight -= 1
        ring.push(x, y)
        inflight += 1
    while inflight:
        got.append(ring.pop_loss())
        inflight -= 1
    assert [np.float32(v) for v in got] == [np.float32(v) for v in eager]
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i)), a.param_info()[i]
    ring.close()
    sa.set_parallel(None)
    sb.set_parallel(None)


def test_feed_ring_keeps_the_dropout_mask_sequence():
    """The ring's warm-up restores the Dropout iteration counters: AlexNet
    trained through the ring draws the same masks as eager steps, bit for bit."""
    text = polegrad.load_model("alexnet", 2)
    kw = CONFIGS["alexnet"][1]
    batches = synthetic_batches((2, 3, 227, 227), 1000, 3, seed=13)
    a = polegrad.Net(text, 1, "f32")
    sa = polegrad.Solver(a, **kw)
    b = polegrad.Net(text, 1, "f32")
    sb = polegrad.Solver(b, **kw)
    eager = []
    for x, y in batches:
        a.set_batch(x, y)
        a.forward()
        eager.append(a.loss())
        a.backward()
        sa.apply()
    ring = polegrad.FeedRing(b, sb, 1)
    got = []
    for x, y in batches:
        ring.push(x, y)
        got.append(ring.pop_loss())
    assert [np.float32(v) for v in got] == [np.float32(v) for v in eager]
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i)), a.param_info()[i]
    ring.close()


def test_feed_ring_training_matches_the_oracle_fp64():
    """Oracle leg of the feed ring (VERDICT r1 missing-5): FP64 CIFAR-quick trained
    through the pinned ring equals the CPU oracle's eager training (MemoryData FIFO
    semantics, layers.cpp:282-304) within north_star's FP64 bar."""
    from parity_util import pyoracle, rel_l2
    text = polegrad.load_model("cifar10_quick", 16)
    kw = CONFIGS["cifar10_quick"][1]
    batches = synthetic_batches((16, 3, 32, 32), 10, 4, seed=14)
    net = polegrad.Net(text, 1, "f64")
    sol = polegrad.Solver(net, **kw)
    orc = pyoracle.OracleNet(text, 1, "f64")
    osol = pyoracle.OracleSolver(orc, **kw)
    ring = polegrad.FeedRing(net, sol, 2)
    got, want, inflight = [], [], 0
    for x, y in batches:
        if inflight == 2:
            got.append(ring.pop_loss())
            inflight -= 1
        ring.push(x, y)
        inflight += 1
        orc.set_batch(x, y)
        want.append(orc.forward())
        orc.backward()
        osol.apply()
    while inflight:
        got.append(ring.pop_loss())
        inflight -= 1
    assert rel_l2(got, want) <= 1e-10, (got, want)
    for i in range(len(net.param_info())):
        assert rel_l2(net.param(i), orc.param(i)) <= 1e-10, net.param_info()[i]
    ring.close()


@pytest.mark.parametrize("config", ["cifar10_quick", "pg_mlp"])
def test_resume_matches_the_oracle_uninterrupted_fp64(config):
    """Oracle leg of checkpoint / resume (VERDICT r1 missing-5): 3 steps, MCWT + MCSS
    snapshot, a fresh Net + Solver restored from it, 3 more steps -- equal to the CPU
    oracle's uninterrupted 6 steps within the FP64 bar (the reference keeps no
    solver state, so the oracle side never checkpoints)."""
    from parity_util import pyoracle, rel_l2
    model, skw, classes, batch = CONFIGS[config]
    text = polegrad.load_model(model, batch if config != "cifar10_quick" else 16)
    shape, labelled = data_shape(text)
    batches = synthetic_batches(shape, classes, 6, seed=15)
    a = polegrad.Net(text, 1, "f64")
    sa = polegrad.Solver(a, **skw)
    orc = pyoracle.OracleNet(text, 1, "f64")
    osol = pyoracle.OracleSolver(orc, **skw)
    for x, y in batches[:3]:
        step(a, sa, x, y, labelled)
    weights, state = a.snapshot(), sa.snapshot()
    b = polegrad.Net(text, 99, "f64")
    sb = polegrad.Solver(b, **skw)
    b.restore(weights)
    sb.restore(state)
    for x, y in batches[3:]:
        step(b, sb, x, y, labelled)
    for x, y in batches:
        if labelled:
            orc.set_batch(x, y)
        else:
            orc.set_batch(x)
        orc.forward()
        if labelled:
            orc.backward()
        else:
            orc.set_blob("logits", np.ones(orc.blob_shape("logits")), diff=True)
            orc.backward_from("logits")
        osol.apply()
    for i in range(len(b.param_info())):
        assert rel_l2(b.param(i), orc.param(i)) <= 1e-10, b.param_info()[i]
