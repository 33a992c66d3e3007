"""Policy-gradient episode on the device: one batched forward
of an episode's states, the modulated log-prob gradients computed on the device
(cdnn_pg_diff) and ONE backward_from(logits) give the same parameter gradients
as the reference trainer's per-step path (trainer.cpp:204-216: batch-1 forward,
pending diff copied into the logits, backward_from, accumulated over the
episode), run here through the unmodified reference Net (oracle)."""
import numpy as np
import pytest

from parity_util import TOL, pyoracle, polegrad, rel_l2

pytestmark = pytest.mark.gpu


def discount(rewards, gamma, normalize):
    """trainer.cpp:64-90 (discount_rewards)"""
    out = np.zeros(len(rewards))
    running = 0.0
    for t in range(len(rewards) - 1, -1, -1):
        running = rewards[t] + gamma * running
        out[t] = running
    if normalize:
        out -= out.mean()
        sd = np.sqrt((out * out).mean())
        if sd >= 1e-10:
            out /= sd
    return out


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("steps", [1, 37, 64])
def test_batched_episode_gradient_matches_per_step_reference(dtype, steps):
    rng = np.random.default_rng(steps)
    states = rng.uniform(-1, 1, (steps, 4, 1, 1))
    rewards = np.ones(steps)
    returns = discount(rewards, 0.99, normalize=True)
    # reference: batch-1 net, one step at a time (the oracle is the unmodified reference Net)
    orc = pyoracle.OracleNet(polegrad.load_model("pg_mlp", 1), 1, dtype)
    actions = np.zeros(steps)
    for t in range(steps):
        orc.set_batch(states[t:t + 1])
        orc.forward()
        p = orc.blob("prob").ravel()
        a = int(rng.uniform() < p[1])  # sampled action
        actions[t] = a
        d = p.copy()
        d[a] -= 1.0
        orc.set_blob("logits", (d * returns[t]).reshape(1, 1, 1, 2), diff=True)
        orc.backward_from("logits")
    # B200: one batch-64 forward of the episode (padded), device diffs, one backward
    net = polegrad.Net(polegrad.load_model("pg_mlp", 64), 1, dtype)
    x = np.zeros((64, 4, 1, 1))
    x[:steps] = states
    net.set_batch(x)
    net.forward()
    net.pg_backward(actions, returns)
    for i, (name, _) in enumerate(net.param_info()):
        err = rel_l2(net.param(i, diff=True), orc.param(i, diff=True))
        assert err <= TOL[dtype], (name, err)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_captured_pg_update_equals_eager(dtype):
    """The captured layer-by-layer episode update (PGStepGraph(fused=False): states / actions / returns H2D, forward,
    device diffs, backward_from, RMSProp, probabilities D2H) replayed on fresh episodes
    trains exactly like the eager Net.pg_backward path, bit for bit."""
    from paper_1810_02272_b200 import cudadnn
    rng = np.random.default_rng(5)
    n, batch = 200, 256
    np_t = np.float64 if dtype == "f64" else np.float32
    episodes = [(rng.uniform(-1, 1, (batch, 4, 1, 1)), np.floor(rng.uniform(0, 1, batch) * 2),
                 rng.standard_normal(batch)) for _ in range(4)]
    text = polegrad.load_model("pg_mlp", batch)
    kw = dict(method="rmsprop", lr=1e-3, rms_decay=0.99, epsilon=1e-8)
    a = polegrad.Net(text, 1, dtype)
    sa = polegrad.Solver(a, **kw)
    b = polegrad.Net(text, 1, dtype)
    sb = polegrad.Solver(b, **kw)
    probs_a = []
    for s, act, ret in episodes:
        a.set_batch(s)
        a.forward()
        a.pg_backward(act[:n], ret[:n])
        sa.apply()
        probs_a.append(a.blob("prob").copy())
    # b: one eager update on the first episode (lazy buffers), then the captured graph
    s, act, ret = episodes[0]
    b.set_batch(s)
    b.forward()
    b.pg_backward(act[:n], ret[:n])
    sb.apply()
    ps, pa, pr = (cudadnn.PinnedBuffer(shape, np_t) for shape in ((batch, 4, 1, 1), (batch,), (batch,)))
    pp = cudadnn.PinnedBuffer((batch, 2), np_t)
    g = polegrad.PGStepGraph(b, sb, ps, pa, pr, n, pp, fused=False)  # the capture applies no update
    assert not g.fused
    for k, (s, act, ret) in enumerate(episodes[1:], start=1):
        ps.array[...] = s
        pa.array[...] = act
        pr.array[...] = ret
        g.replay()
        b.sync()
        assert np.array_equal(pp.array.reshape(probs_a[k].shape), probs_a[k].astype(np_t))
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i)), a.param_info()[i]


def _episodes(rng, count, batch):
    return [(rng.uniform(-1, 1, (batch, 4, 1, 1)), np.floor(rng.uniform(0, 1, batch) * 2), rng.standard_normal(batch))
            for _ in range(count)]


FUSED_CASES = [("f64", dict(method="rmsprop", lr=1e-3, rms_decay=0.99, epsilon=1e-8)),
               ("f64", dict(method="sgd", lr=1e-2, momentum=0.9, weight_decay=1e-3)),
               ("f32", dict(method="sgd", lr=1e-2, momentum=0.9, weight_decay=1e-3)),
               ("f32", dict(method="sgd", lr=1e-3))]


@pytest.mark.parametrize("dtype,kw", FUSED_CASES)
@pytest.mark.parametrize("batch,n", [(1024, 1024), (256, 200), (2500, 1999)])
def test_fused_pg_update_matches_eager_and_oracle(dtype, kw, batch, n):
    """The pg_softmax MLP's captured update is ONE kernel (cdnn_mlp_pg_step: forward,
    softmax gradient of the first n rows, backward, the solver rule).  Replayed on
    fresh episodes it trains like the eager layered path (Net.pg_backward + Solver)
    and like the unmodified reference Net + solver (oracle) to the parity bar: the
    same operations summed in another order.  batch 2500 takes three row passes."""
    from paper_1810_02272_b200 import cudadnn
    rng = np.random.default_rng(batch + n)
    np_t = np.float64 if dtype == "f64" else np.float32
    eps = _episodes(rng, 4, batch)
    text = polegrad.load_model("pg_mlp", batch)
    a = polegrad.Net(text, 1, dtype)
    sa = polegrad.Solver(a, **kw)
    b = polegrad.Net(text, 1, dtype)
    sb = polegrad.Solver(b, **kw)
    orc = pyoracle.OracleNet(text, 1, dtype)
    so = pyoracle.OracleSolver(orc, **kw)
    for i in range(len(a.param_info())):  # same initial weights everywhere
        orc.set_param(i, a.param(i))
        assert np.array_equal(a.param(i), b.param(i))
    probs_a, probs_o = [], []
    for s, act, ret in eps:
        a.set_batch(s)
        a.forward()
        a.pg_backward(act[:n], ret[:n])
        sa.apply()
        probs_a.append(a.blob("prob").copy())
        orc.set_batch(s)
        orc.forward()
        p = orc.blob("prob").reshape(batch, 2)
        d = np.zeros_like(p)
        d[:n] = p[:n]
        d[np.arange(n), act[:n].astype(int)] -= 1.0
        d[:n] *= ret[:n, None]
        orc.set_blob("logits", d.reshape(batch, 2, 1, 1), diff=True)
        orc.backward_from("logits")
        so.apply()
        probs_o.append(p.copy())
    s, act, ret = eps[0]
    b.set_batch(s)
    b.forward()
    b.pg_backward(act[:n], ret[:n])
    sb.apply()
    ps, pa, pr = (cudadnn.PinnedBuffer(shape, np_t) for shape in ((batch, 4, 1, 1), (batch,), (batch,)))
    pp = cudadnn.PinnedBuffer((batch, 2), np_t)
    g = polegrad.PGStepGraph(b, sb, ps, pa, pr, n, pp)
    assert g.fused
    tol = 1e-10 if dtype == "f64" else TOL["f32"]
    for k, (s, act, ret) in enumerate(eps[1:], start=1):
        ps.array[...] = s
        pa.array[...] = act
        pr.array[...] = ret
        g.replay()
        b.sync()
        got = pp.array.reshape(batch, 2).astype(np.float64)
        assert rel_l2(got, probs_a[k]) <= tol, ("prob vs eager", k)
        assert rel_l2(got, probs_o[k]) <= tol, ("prob vs oracle", k)
    for i, (name, _) in enumerate(a.param_info()):
        wb = b.param(i)
        assert rel_l2(wb, a.param(i)) <= tol, (name, "vs eager")
        assert rel_l2(wb, orc.param(i)) <= tol, (name, "vs oracle")
        assert not np.any(b.param(i, diff=True)), (name, "gradient left non-zero")
