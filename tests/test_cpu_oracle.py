"""Pinning the CPU oracle (no GPU needed).

* The reference part of the oracle IS the unmodified reference (its own unit
  suite passes, test_cpu_reference_suite.py); here: its published known-answer
  values through the oracle driver, and ExtNet == reference Net bit for bit.
* The extension layers (absent from the reference) against torch float64 and
  central finite differences."""
import numpy as np
import pytest
import torch

from parity_util import pyoracle, rel_l2

pytestmark = pytest.mark.skipif(not pyoracle.available("f64"), reason="oracle/_ref not built")


def test_gemm_known_answers():
    # backend_test.cpp:173-182: [[1,2],[3,4]] * [1,1]^T = [3,7]
    c = pyoracle.reference_gemm(0, 0, 2, 1, 2, 1.0, [1, 2, 3, 4], [1, 1], 0.0, [np.nan, np.nan])
    assert c.tolist() == [3.0, 7.0]
    rng = np.random.default_rng(0)
    for ta in (0, 1):
        for tb in (0, 1):
            m, n, k = 5, 7, 3
            A = rng.uniform(-1, 1, (k, m) if ta else (m, k))
            B = rng.uniform(-1, 1, (n, k) if tb else (k, n))
            C0 = rng.uniform(-1, 1, (m, n))
            got = pyoracle.reference_gemm(ta, tb, m, n, k, 0.5, A, B, 0.25, C0)
            want = 0.5 * (A.T if ta else A) @ (B.T if tb else B) + 0.25 * C0
            assert np.allclose(got.reshape(m, n), want, rtol=1e-12, atol=1e-12)


def test_extension_net_matches_reference_net_bit_exact():
    from paper_1810_02272_b200 import polegrad
    text = polegrad.load_model("pg_mlp")
    a = pyoracle.OracleNet(text, 1, "f64", reference=True)
    b = pyoracle.OracleNet(text, 1, "f64", reference=False)
    assert a.kind == "reference" and b.kind == "extension"
    rng = np.random.default_rng(1)
    x = rng.uniform(-1, 1, (1024, 4))
    g = rng.uniform(-1, 1, (1024, 2))
    sa = pyoracle.OracleSolver(a, "rmsprop", 1e-3)
    sb = pyoracle.OracleSolver(b, "rmsprop", 1e-3)
    for _ in range(3):
        for n in (a, b):
            n.set_batch(x)
            n.forward()
            n.set_blob("logits", g, diff=True)
            n.backward_from("logits")
        assert np.array_equal(a.blob("prob"), b.blob("prob"))
        for i in range(4):
            assert np.array_equal(a.param(i, True), b.param(i, True))
        sa.apply()
        sb.apply()
    assert a.snapshot() == b.snapshot()


def conv_net(n, c, h, w, co, k, s, p, g=1):
    # data -> convA (3x3 same, gives convB a bottom that needs a gradient) -> convB
    return f"""
layer {{ name: "d" type: "MemoryData" top: "x" memory_data_param {{ batch_size: {n} channels: {c} height: {h} width: {w} }} }}
layer {{ name: "a" type: "Convolution" bottom: "x" top: "a" convolution_param {{ num_output: {c} kernel_size: 1 }} }}
layer {{ name: "b" type: "Convolution" bottom: "a" top: "b"
  convolution_param {{ num_output: {co} kernel_size: {k} stride: {s} pad: {p} group: {g} }} }}
"""


@pytest.mark.parametrize("case", [(2, 3, 9, 9, 4, 3, 1, 1, 1), (2, 4, 11, 10, 6, 5, 2, 2, 2), (1, 2, 7, 7, 3, 7, 1, 0, 1)])
def test_convolution_extension_vs_torch(case):
    n, c, h, w, co, k, s, p, g = case
    net = pyoracle.OracleNet(conv_net(n, c, h, w, co, k, s, p, g), 3, "f64")
    rng = np.random.default_rng(sum(case))
    x = rng.uniform(-1, 1, (n, c, h, w))
    net.set_batch(x)
    net.forward()
    a = torch.from_numpy(net.blob("a")).requires_grad_()
    wb = torch.from_numpy(net.param(2)).requires_grad_()
    bb = torch.from_numpy(net.param(3).ravel()).requires_grad_()
    y = torch.nn.functional.conv2d(a, wb, bb, stride=s, padding=p, groups=g)
    assert rel_l2(net.blob("b"), y.detach().numpy()) < 1e-13
    dy = rng.uniform(-1, 1, tuple(y.shape))
    y.backward(torch.from_numpy(dy))
    net.set_blob("b", dy, diff=True)
    net.backward()
    assert rel_l2(net.param(2, True), wb.grad.numpy()) < 1e-13
    assert rel_l2(net.param(3, True).ravel(), bb.grad.numpy()) < 1e-13
    assert rel_l2(net.blob("a", True), a.grad.numpy()) < 1e-13
    # data does not need a gradient: the first convolution skips backward-data (Caffe propagate_down)
    assert not net.blob("x", True).any()


@pytest.mark.parametrize("method", ["MAX", "AVE"])
@pytest.mark.parametrize("geom", [(24, 24, 2, 2, 0), (32, 32, 3, 2, 0), (13, 11, 3, 2, 1), (8, 8, 3, 3, 1)])
def test_pooling_extension(method, geom):
    h, w, k, s, p = geom
    text = f"""
layer {{ name: "d" type: "MemoryData" top: "x" memory_data_param {{ batch_size: 2 channels: 3 height: {h} width: {w} }} }}
layer {{ name: "c" type: "Convolution" bottom: "x" top: "c" convolution_param {{ num_output: 3 kernel_size: 1 }} }}
layer {{ name: "p" type: "Pooling" bottom: "c" top: "y" pooling_param {{ pool: {method} kernel_size: {k} stride: {s} pad: {p} }} }}
"""
    net = pyoracle.OracleNet(text, 1, "f64")
    x = np.random.default_rng(h * w + k).standard_normal((2, 3, h, w))
    net.set_batch(x)
    net.forward()
    c = net.blob("c")
    ct = torch.from_numpy(c).requires_grad_()
    if method == "MAX":
        yt, idx = torch.nn.functional.max_pool2d(ct, k, s, p, ceil_mode=True, return_indices=True)
        mask = net.pool_mask("p", int(np.prod(yt.shape)))
        # torch flat indices are h*W+w within the plane as well
        assert np.array_equal(mask, idx.numpy().ravel().astype(np.int32))
    else:
        # Caffe AVE: divisor counts padding but not the overhang past H+pad
        yt = torch.nn.functional.avg_pool2d(ct, k, s, p, ceil_mode=True, count_include_pad=True)
        if p:  # torch's ceil-mode edge divisor differs from Caffe's; restate Caffe directly
            yt = torch.from_numpy(caffe_ave_pool(c, k, s, p, net.blob_shape("y"))).requires_grad_()
    assert net.blob_shape("y") == tuple(yt.shape)
    assert rel_l2(net.blob("y"), yt.detach().numpy()) < 1e-13
    if method == "MAX" or not p:
        dy = np.random.default_rng(5).standard_normal(tuple(yt.shape))
        yt.backward(torch.from_numpy(dy))
        net.set_blob("y", dy, diff=True)
        net.backward()
        assert rel_l2(net.blob("c", True), ct.grad.numpy()) < 1e-13


def caffe_ave_pool(x, k, s, p, shape):
    n, c, h, w = x.shape
    _, _, ph_, pw_ = shape
    y = np.zeros(shape)
    for i in range(ph_):
        for j in range(pw_):
            hs, ws = i * s - p, j * s - p
            he, we = min(hs + k, h + p), min(ws + k, w + p)
            size = (he - hs) * (we - ws)
            hs, ws, he, we = max(hs, 0), max(ws, 0), min(he, h), min(we, w)
            y[:, :, i, j] = x[:, :, hs:he, ws:we].sum(axis=(2, 3)) / size
    return y


def test_softmax_with_loss_extension():
    text = """
layer { name: "d" type: "MemoryData" top: "x" top: "label" memory_data_param { batch_size: 16 channels: 10 height: 1 width: 1 } }
layer { name: "ip" type: "InnerProduct" bottom: "x" top: "s" inner_product_param { num_output: 10 } }
layer { name: "loss" type: "SoftmaxWithLoss" bottom: "s" bottom: "label" top: "loss" }
"""
    net = pyoracle.OracleNet(text, 1, "f64")
    rng = np.random.default_rng(2)
    x = rng.uniform(-1, 1, (16, 10, 1, 1))
    lab = rng.integers(0, 10, 16).astype(np.float64)
    net.set_batch(x, lab)
    loss = net.forward()
    s = torch.from_numpy(net.blob("s").reshape(16, 10)).requires_grad_()
    lt = torch.nn.functional.cross_entropy(s, torch.from_numpy(lab.astype(np.int64)))
    lt.backward()
    assert abs(loss - lt.item()) < 1e-13
    net.backward()
    assert rel_l2(net.blob("s", True).reshape(16, 10), s.grad.numpy()) < 1e-13


def test_split_sums_fanout_gradients():
    # x feeds two InnerProducts: the automatic Split must SUM their input gradients
    text = """
layer { name: "d" type: "MemoryData" top: "x" memory_data_param { batch_size: 3 channels: 4 height: 1 width: 1 } }
layer { name: "pre" type: "InnerProduct" bottom: "x" top: "h" inner_product_param { num_output: 5 } }
layer { name: "a" type: "InnerProduct" bottom: "h" top: "ya" inner_product_param { num_output: 2 } }
layer { name: "b" type: "InnerProduct" bottom: "h" top: "yb" inner_product_param { num_output: 2 } }
"""
    net = pyoracle.OracleNet(text, 1, "f64", reference=False)
    rng = np.random.default_rng(4)
    net.set_batch(rng.uniform(-1, 1, (3, 4, 1, 1)))
    net.forward()
    ga, gb = rng.uniform(-1, 1, (3, 1, 1, 2)), rng.uniform(-1, 1, (3, 1, 1, 2))
    net.set_blob("ya", ga, diff=True)
    net.set_blob("yb", gb, diff=True)
    net.backward()
    wa, wb = net.param(2).reshape(2, 5), net.param(4).reshape(2, 5)
    want = ga.reshape(3, 2) @ wa + gb.reshape(3, 2) @ wb
    assert rel_l2(net.blob("h", True).reshape(3, 5), want) < 1e-14


def test_cifar_quick_finite_differences():
    """Central differences (the reference FD recipe, gradient_check.hpp:14-82) on a
    batch-2 CIFAR-quick, objective = loss, a sample of weights per layer."""
    from paper_1810_02272_b200 import polegrad
    text = polegrad.load_model("cifar10_quick").replace("batch_size: 100", "batch_size: 2")
    net = pyoracle.OracleNet(text, 1, "f64")
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, 3, 32, 32))
    y = np.array([3.0, 7.0])

    def loss():
        net.set_batch(x, y)
        return net.forward()

    loss()
    net.backward()
    eps = 1e-5
    for i, (name, shape) in enumerate(net.param_info()):
        w = net.param(i)
        g = net.param(i, True).ravel()
        flat = w.ravel().copy()
        for j in rng.choice(flat.size, size=min(4, flat.size), replace=False):
            for sgn, store in ((1, "p"), (-1, "m")):
                f2 = flat.copy()
                f2[j] += sgn * eps
                net.set_param(i, f2.reshape(shape))
                if store == "p":
                    lp = loss()
                else:
                    lm = loss()
            net.set_param(i, w)
            num = (lp - lm) / (2 * eps)
            err = abs(num - g[j]) / max(abs(num), abs(g[j]), 1e-8)
            assert err < 1e-4 or abs(num - g[j]) < 1e-9, (name, j, num, g[j])
