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
    """The captured episode update (PGStepGraph: states / actions / returns H2D, forward,
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
    g = polegrad.PGStepGraph(b, sb, ps, pa, pr, n, pp)  # the capture itself applies no update
    for k, (s, act, ret) in enumerate(episodes[1:], start=1):
        ps.array[...] = s
        pa.array[...] = act
        pr.array[...] = ret
        g.replay()
        b.sync()
        assert np.array_equal(pp.array.reshape(probs_a[k].shape), probs_a[k].astype(np_t))
    for i in range(len(a.param_info())):
        assert np.array_equal(a.param(i), b.param(i)), a.param_info()[i]
