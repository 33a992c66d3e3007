"""Pinning the oracle's restatement of the config-4/5 layers (LRN, Dropout,
BatchNorm, Scale, Eltwise — absent from the reference)
against torch float64 and central finite differences.  CPU only."""
import numpy as np
import pytest
import torch

from parity_util import pyoracle, rel_l2

MASK64 = (1 << 64) - 1


def data_layer(n, c, h, w):
    return (f'layer {{ name: "d" type: "MemoryData" top: "x" memory_data_param {{ batch_size: {n} channels: {c} '
            f'height: {h} width: {w} }} }}\n'
            # a 1x1 conv gives the layer under test a bottom that needs a gradient
            f'layer {{ name: "a" type: "Convolution" bottom: "x" top: "a" convolution_param {{ num_output: {c} '
            f'kernel_size: 1 }} }}\n')


def run(text, x, top, dy_seed=7):
    net = pyoracle.OracleNet(text, 3, "f64")
    net.set_batch(x)
    net.forward()
    a = net.blob("a")
    y = net.blob(top)
    dy = np.random.default_rng(dy_seed).uniform(-1, 1, y.shape)
    net.set_blob(top, dy, diff=True)
    net.backward()
    return net, a, y, dy


@pytest.mark.parametrize("size,alpha,beta,k", [(5, 1e-4, 0.75, 1.0), (3, 0.5, 0.75, 2.0), (5, 2.0, 0.5, 1.0)])
def test_lrn_vs_torch(size, alpha, beta, k):
    n, c, h, w = 2, 7, 5, 4
    text = data_layer(n, c, h, w) + (f'layer {{ name: "l" type: "LRN" bottom: "a" top: "y" lrn_param {{ '
                                     f'local_size: {size} alpha: {alpha} beta: {beta} k: {k} }} }}\n')
    x = np.random.default_rng(1).uniform(-2, 2, (n, c, h, w))
    net, a, y, dy = run(text, x, "y")
    ta = torch.from_numpy(a).requires_grad_()
    ty = torch.nn.functional.local_response_norm(ta, size, alpha=alpha, beta=beta, k=k)
    ty.backward(torch.from_numpy(dy))
    assert rel_l2(y, ty.detach().numpy()) < 1e-13
    assert rel_l2(net.blob("a", True), ta.grad.numpy()) < 1e-12


def np_drop_hash(seed, it, idx):
    """numpy restatement of the counter hash (ops_layers.cu drop_hash)."""
    with np.errstate(over="ignore"):
        z = (np.uint64(seed) * np.uint64(0x9E3779B97F4A7C15)) ^ (np.uint64(it + 1) * np.uint64(0xBF58476D1CE4E5B9)) \
            ^ ((idx.astype(np.uint64) + np.uint64(1)) * np.uint64(0x94D049BB133111EB))
        z ^= z >> np.uint64(30)
        z *= np.uint64(0xBF58476D1CE4E5B9)
        z ^= z >> np.uint64(27)
        z *= np.uint64(0x94D049BB133111EB)
        z ^= z >> np.uint64(31)
    return (z >> np.uint64(32)).astype(np.uint32)


@pytest.mark.parametrize("ratio", [0.5, 0.2])
def test_dropout_mask_and_scaling(ratio):
    n, c, h, w = 4, 3, 8, 8
    text = data_layer(n, c, h, w) + (f'layer {{ name: "dr" type: "Dropout" bottom: "a" top: "y" dropout_param {{ '
                                     f'dropout_ratio: {ratio} }} }}\n')
    x = np.random.default_rng(2).uniform(0.5, 1.5, (n, c, h, w))  # nonzero so the mask is visible
    net, a, y, dy = run(text, x, "y")
    keep = y != 0
    # kept values scaled by 1/(1-ratio), dropped are zero; gradient uses the same mask
    assert np.allclose(y[keep], a[keep] / (1 - ratio), rtol=1e-15)
    da = net.blob("a", True)
    assert np.array_equal(da != 0, keep)
    assert np.allclose(da[keep], dy[keep] / (1 - ratio), rtol=1e-15)
    # the mask is the counter hash of (seed, iteration 1, index) for some seed: recover the
    # threshold relation on the hash values (kept iff hash > ratio * 2^32)
    frac = keep.mean()
    assert abs(frac - (1 - ratio)) < 0.08
    # a second forward draws a different mask (iteration counter advanced)
    net.set_batch(x)
    net.forward()
    assert not np.array_equal(net.blob("y") != 0, keep)


def test_dropout_hash_matches_numpy_restatement():
    """The oracle's mask is exactly {hash(seed, 1, i) > ratio*2^32}: find the seed by
    taking the layer's first Rng draw (the net seed's mt19937_64 stream after the 1x1
    conv's weights) through a one-parameter-free net: Dropout directly on the data."""
    n, c, h, w = 2, 2, 4, 4
    ratio = 0.5
    text = (f'layer {{ name: "d" type: "MemoryData" top: "x" memory_data_param {{ batch_size: {n} channels: {c} '
            f'height: {h} width: {w} }} }}\n'
            f'layer {{ name: "dr" type: "Dropout" bottom: "x" top: "y" dropout_param {{ dropout_ratio: {ratio} }} }}\n')
    seed = 11
    net = pyoracle.OracleNet(text, seed, "f64")
    x = np.ones((n, c, h, w))
    net.set_batch(x)
    net.forward()
    keep = (net.blob("y") != 0).ravel()
    # mt19937_64 first output for `seed` (std::mt19937_64, the reference Rng engine)
    first = _mt19937_64_first(seed)
    thr = np.uint32(int(ratio * 2 ** 32))
    want = np_drop_hash(first, 1, np.arange(n * c * h * w)) > thr
    assert np.array_equal(keep, want)


def _mt19937_64_first(seed):
    """First output of std::mt19937_64(seed) (pure Python, for the hash test)."""
    nn, mm = 312, 156
    mt = [0] * nn
    mt[0] = seed & MASK64
    for i in range(1, nn):
        mt[i] = (6364136223846793005 * (mt[i - 1] ^ (mt[i - 1] >> 62)) + i) & MASK64
    upper, lower = 0xFFFFFFFF80000000, 0x7FFFFFFF
    mag = [0, 0xB5026F5AA96619E9]
    x = (mt[0] & upper) | (mt[1] & lower)
    y = mt[mm] ^ (x >> 1) ^ mag[x & 1]
    y ^= (y >> 29) & 0x5555555555555555
    y ^= (y << 17) & 0x71D67FFFEDA60000
    y ^= (y << 37) & 0xFFF7EEE000000000
    y ^= y >> 43
    return y & MASK64


@pytest.mark.parametrize("shape", [(4, 3, 5, 5), (8, 16, 4, 4), (3, 2, 1, 1)])
def test_batchnorm_vs_torch(shape):
    text = data_layer(*shape) + 'layer { name: "bn" type: "BatchNorm" bottom: "a" top: "y" }\n'
    x = np.random.default_rng(3).uniform(-1, 3, shape)
    net, a, y, dy = run(text, x, "y")
    ta = torch.from_numpy(a).requires_grad_()
    ty = torch.nn.functional.batch_norm(ta, None, None, training=True, eps=1e-5)
    ty.backward(torch.from_numpy(dy))
    assert rel_l2(y, ty.detach().numpy()) < 1e-12
    assert rel_l2(net.blob("a", True), ta.grad.numpy()) < 1e-10


@pytest.mark.parametrize("bias", [True, False])
def test_scale_vs_torch(bias):
    n, c, h, w = 3, 4, 3, 5
    text = data_layer(n, c, h, w) + (f'layer {{ name: "s" type: "Scale" bottom: "a" top: "y" scale_param {{ '
                                     f'bias_term: {"true" if bias else "false"} }} }}\n')
    net = pyoracle.OracleNet(text, 3, "f64")
    rng = np.random.default_rng(4)
    gamma = rng.uniform(0.5, 1.5, (1, 1, 1, c))
    net.set_param(2, gamma)
    if bias:
        net.set_param(3, rng.uniform(-1, 1, (1, 1, 1, c)))
    x = rng.uniform(-1, 1, (n, c, h, w))
    net.set_batch(x)
    net.forward()
    a = net.blob("a")
    tg = torch.from_numpy(net.param(2).reshape(c)).requires_grad_()
    tb = torch.from_numpy(net.param(3).reshape(c)).requires_grad_() if bias else None
    ta = torch.from_numpy(a).requires_grad_()
    ty = ta * tg[None, :, None, None] + (tb[None, :, None, None] if bias else 0)
    assert rel_l2(net.blob("y"), ty.detach().numpy()) < 1e-15
    dy = rng.uniform(-1, 1, (n, c, h, w))
    ty.backward(torch.from_numpy(dy))
    net.set_blob("y", dy, diff=True)
    net.backward()
    assert rel_l2(net.param(2, True).reshape(c), tg.grad.numpy()) < 1e-13
    if bias:
        assert rel_l2(net.param(3, True).reshape(c), tb.grad.numpy()) < 1e-13
    assert rel_l2(net.blob("a", True), ta.grad.numpy()) < 1e-14


def test_eltwise_sum_with_coefficients_and_fanout():
    # y = 2*a + (-0.5)*b with a = conv(x), b = conv(a): a fans out (Split), its gradient sums both paths
    text = data_layer(2, 3, 4, 4) + """
layer { name: "b" type: "Convolution" bottom: "a" top: "b" convolution_param { num_output: 3 kernel_size: 3 pad: 1 } }
layer { name: "e" type: "Eltwise" bottom: "a" bottom: "b" top: "y" eltwise_param { operation: SUM coeff: 2 coeff: -0.5 } }
"""
    x = np.random.default_rng(5).uniform(-1, 1, (2, 3, 4, 4))
    net, a, y, dy = run(text, x, "y")
    ta = torch.from_numpy(a).requires_grad_()
    wb = torch.from_numpy(net.param(2))
    bb = torch.from_numpy(net.param(3).ravel())
    tb = torch.nn.functional.conv2d(ta, wb, bb, padding=1)
    ty = 2 * ta - 0.5 * tb
    assert rel_l2(y, ty.detach().numpy()) < 1e-14
    ty.backward(torch.from_numpy(dy))
    assert rel_l2(net.blob("a", True), ta.grad.numpy()) < 1e-13


def test_inplace_bn_scale_relu_chain_matches_out_of_place():
    """conv -> BN -> Scale -> ReLU all in place == the same net with distinct tops."""
    base = data_layer(4, 3, 6, 6)
    inplace = base + """
layer { name: "bn" type: "BatchNorm" bottom: "a" top: "a" }
layer { name: "sc" type: "Scale" bottom: "a" top: "a" scale_param { bias_term: true } }
layer { name: "r" type: "ReLU" bottom: "a" top: "a" }
layer { name: "c" type: "Convolution" bottom: "a" top: "y" convolution_param { num_output: 2 kernel_size: 3 } }
"""
    distinct = base + """
layer { name: "bn" type: "BatchNorm" bottom: "a" top: "b1" }
layer { name: "sc" type: "Scale" bottom: "b1" top: "b2" scale_param { bias_term: true } }
layer { name: "r" type: "ReLU" bottom: "b2" top: "b3" }
layer { name: "c" type: "Convolution" bottom: "b3" top: "y" convolution_param { num_output: 2 kernel_size: 3 } }
"""
    x = np.random.default_rng(6).uniform(-1, 1, (4, 3, 6, 6))
    n1, _, y1, _ = run(inplace, x, "y")
    n2, _, y2, _ = run(distinct, x, "y")
    assert np.array_equal(y1, y2)
    for i in range(len(n1.param_info())):
        assert np.array_equal(n1.param(i, True), n2.param(i, True)), i


def test_resnet8_finite_differences():
    """Central differences on a batch-2 ResNet-8 (same generator as ResNet-20, one
    block per stage): BatchNorm, Scale, Eltwise, projection shortcut, global pooling."""
    from paper_1810_02272_b200.models.gen_resnet import resnet
    text = resnet(8, batch=2)
    net = pyoracle.OracleNet(text, 1, "f64")
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, 3, 32, 32))
    y = np.array([3.0, 7.0])

    def loss():
        net.set_batch(x, y)
        return net.forward()

    loss()
    net.backward()
    eps = 1e-7  # small: ~30k ReLU inputs per layer, a 1e-5 step crosses kinks
    info = net.param_info()
    for i in range(0, len(info), 3):
        name, shape = info[i]
        w = net.param(i)
        g = net.param(i, True).ravel()
        flat = w.ravel().copy()
        for j in rng.choice(flat.size, size=min(2, flat.size), replace=False):
            vals = []
            for sgn in (1, -1):
                f2 = flat.copy()
                f2[j] += sgn * eps
                net.set_param(i, f2.reshape(shape))
                vals.append(loss())
            net.set_param(i, w)
            num = (vals[0] - vals[1]) / (2 * eps)
            err = abs(num - g[j]) / max(abs(num), abs(g[j]), 1e-8)
            assert err < 1e-4 or abs(num - g[j]) < 1e-7, (name, j, num, g[j])
