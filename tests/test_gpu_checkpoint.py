"""Checkpoint / resume: MCWT weights + MCSS solver state
taken mid-run restore into a fresh Net and Solver, and the resumed run is bit
identical to the uninterrupted one (same kernels, deterministic reductions)."""
import numpy as np
import pytest

from parity_util import CONFIGS, data_shape, polegrad, synthetic_batches

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
