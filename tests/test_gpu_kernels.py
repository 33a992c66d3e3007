"""Numerics of the sm_100a kernels behind the C-ABI against fp64 references.

TF32 tolerance: the float path feeds the tensor cores TF32 (10-bit mantissa,
inputs rounded to nearest), accumulates in fp32; relative L2 error of a GEMM
is ~1e-4..1e-3, so float checks use rel-L2 <= 2e-3 (north_star's TF32 bar);
FP64 checks use 1e-12.
"""
import ctypes as C
import numpy as np
import pytest
import torch

from paper_1810_02272_b200 import cudadnn as cd

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


TOL = {cd.F32: 2e-3, cd.F64: 1e-12}
NP = {cd.F32: np.float32, cd.F64: np.float64}


@pytest.fixture(params=["tf32x3", "tf32"])
def math(request, ctx):
    """Both float numerics modes; 3xTF32 (the default) must also reach ~fp32 accuracy."""
    mode = cd.MATH_TF32X3 if request.param == "tf32x3" else cd.MATH_TF32
    ctx.call("cdnn_set_math_mode", mode)
    yield request.param
    ctx.call("cdnn_set_math_mode", cd.MATH_TF32X3)


def test_tf32x3_reaches_fp32_accuracy(ctx):
    rng = np.random.default_rng(11)
    m, n, k = 256, 192, 2048
    A = rng.standard_normal((m, k)).astype(np.float32)
    B = rng.standard_normal((k, n)).astype(np.float32)
    want = A.astype(np.float64) @ B.astype(np.float64)
    errs = {}
    for name, mode in (("tf32x3", cd.MATH_TF32X3), ("tf32", cd.MATH_TF32)):
        ctx.call("cdnn_set_math_mode", mode)
        ha, hb, hc = ctx.upload(A), ctx.upload(B), ctx.alloc(m * n, cd.F32)
        ctx.call("cdnn_gemm", 0, 0, m, n, k, 1.0, ha, hb, 0.0, hc, 0)
        errs[name] = rel_l2(ctx.read(hc), want)
    ctx.call("cdnn_set_math_mode", cd.MATH_TF32X3)
    assert errs["tf32x3"] < 2e-6, errs      # fp32-level
    assert errs["tf32"] < 2e-3, errs        # plain tf32
    assert errs["tf32x3"] < errs["tf32"] / 50, errs


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(2, 1, 2), (64, 500, 800), (100, 64, 1024), (37, 19, 300), (256, 128, 96),
                                   (1024, 2, 10), (300, 260, 4100), (2, 10, 1024), (10, 4, 2048)])
def test_gemm(ctx, math, dtype, ta, tb, m, n, k):
    rng = np.random.default_rng(m * 7 + n * 3 + k)
    A = rng.uniform(-1, 1, (k, m) if ta else (m, k))
    B = rng.uniform(-1, 1, (n, k) if tb else (k, n))
    Cin = rng.uniform(-1, 1, (m, n))
    alpha, beta = 0.5, 0.25
    ha, hb, hc = ctx.upload(A.astype(NP[dtype])), ctx.upload(B.astype(NP[dtype])), ctx.upload(Cin.astype(NP[dtype]))
    ctx.call("cdnn_gemm", ta, tb, m, n, k, alpha, ha, hb, beta, hc, 0)
    got = ctx.read(hc).reshape(m, n)
    opA = A.T if ta else A
    opB = B.T if tb else B
    want = alpha * opA.astype(NP[dtype]).astype(np.float64) @ opB.astype(NP[dtype]).astype(np.float64) + beta * Cin.astype(NP[dtype])
    assert rel_l2(got, want) <= TOL[dtype]
    for h in (ha, hb, hc):
        ctx.free(h)


def test_gemm_beta_zero_ignores_nan(ctx):
    A = np.array([[1, 2], [3, 4]], np.float32)
    B = np.array([[1], [1]], np.float32)
    hc = ctx.upload(np.full(2, np.nan, np.float32))
    ha, hb = ctx.upload(A), ctx.upload(B)
    ctx.call("cdnn_gemm", 0, 0, 2, 1, 2, 1.0, ha, hb, 0.0, hc, 0)
    assert ctx.read(hc).tolist() == [3.0, 7.0]


def conv_ref(x, w, b, stride, pad, dil, group):
    t = torch.nn.functional.conv2d(torch.from_numpy(x), torch.from_numpy(w), torch.from_numpy(b) if b is not None else None,
                                   stride=stride, padding=pad, dilation=dil, groups=group)
    return t.numpy()


CONV_CASES = [
    # n, c, h, w, co, k, stride, pad, dil, group
    (4, 1, 28, 28, 20, 5, 1, 0, 1, 1),      # LeNet conv1
    (4, 20, 12, 12, 50, 5, 1, 0, 1, 1),     # LeNet conv2
    (3, 3, 32, 32, 32, 5, 1, 2, 1, 1),      # CIFAR-quick conv1
    (2, 32, 16, 16, 32, 5, 1, 2, 1, 1),     # CIFAR-quick conv2
    (2, 32, 8, 8, 64, 5, 1, 2, 1, 1),       # CIFAR-quick conv3
    (2, 3, 35, 35, 16, 11, 4, 0, 1, 1),     # AlexNet conv1 shape (small)
    (2, 2, 31, 30, 16, 7, 2, 3, 1, 1),      # space-to-depth stem: padded, ragged, s = 2
    (2, 1, 37, 40, 16, 9, 8, 1, 1, 1),      # space-to-depth stem: s = 8 phases per input row
    (2, 8, 13, 13, 12, 3, 1, 1, 1, 2),      # grouped
    (2, 16, 15, 15, 32, 3, 2, 1, 1, 1),     # ResNet downsample
    (2, 4, 9, 9, 8, 3, 1, 2, 2, 1),         # dilation
    (2, 96, 13, 13, 64, 3, 1, 1, 1, 1),     # three 32-channel blocks (tap-shift kernel, double-buffered A)
    (2, 48, 27, 27, 64, 5, 1, 2, 1, 2),     # AlexNet conv2 shape, grouped, 24 channels per group
    (4, 16, 32, 32, 16, 3, 1, 1, 1, 1),     # ResNet-20 stage 1
    (2, 64, 8, 8, 32, 1, 1, 0, 1, 1),       # 1x1
    (1, 64, 13, 13, 256, 3, 1, 1, 1, 1),    # two 128-wide output blocks
    (2, 8, 12, 10, 8, 3, 1, 0, 3, 1),       # dilation 3, no padding
    (2, 3, 39, 39, 96, 11, 4, 0, 1, 1),     # AlexNet conv1 (96 outputs: N = 96 tiles)
    (2, 96, 15, 15, 256, 5, 1, 2, 1, 2),    # AlexNet conv2 (backward-data to 48 channels: N = 48 tiles)
    (2, 384, 13, 13, 384, 3, 1, 1, 1, 2),   # AlexNet conv4 (192 per group: N = 96 tiles)
    (100, 32, 16, 16, 32, 5, 1, 2, 1, 1),   # CIFAR-quick conv2 at bench size (split-K clusters of 8 CTAs)
    (64, 16, 32, 32, 16, 3, 1, 1, 1, 1),    # ResNet-20 stage 1, half the bench batch
    (3, 96, 9, 9, 64, 1, 1, 0, 1, 1),       # dual MMA issuers, one-tap blocks: the issuers alternate blocks
    (5, 32, 13, 13, 64, 3, 1, 1, 1, 1),     # dual MMA issuers, 3 ring stages per tile: parity alternates per tile
]


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("case", CONV_CASES)
def test_conv(ctx, math, dtype, case):
    n, c, h, w, co, k, s, p, dl, g = case
    rng = np.random.default_rng(sum(case))
    x = rng.uniform(-1, 1, (n, c, h, w))
    wt = rng.uniform(-1, 1, (co, c // g, k, k))
    b = rng.uniform(-1, 1, co)
    y = conv_ref(x, wt, b, s, p, dl, g)
    dy = rng.uniform(-1, 1, y.shape)
    xt = torch.from_numpy(x).requires_grad_()
    wtt = torch.from_numpy(wt).requires_grad_()
    bt = torch.from_numpy(b).requires_grad_()
    yt = torch.nn.functional.conv2d(xt, wtt, bt, stride=s, padding=p, dilation=dl, groups=g)
    yt.backward(torch.from_numpy(dy))
    dt = NP[dtype]
    d = ctx.conv_desc(n, c, h, w, co, k, s, p, dl, g)
    assert ctx.conv_output_shape(d) == y.shape
    hx, hw, hb = ctx.upload(x.astype(dt)), ctx.upload(wt.astype(dt)), ctx.upload(b.astype(dt))
    hy = ctx.alloc(y.size, dtype)
    ctx.call("cdnn_conv_forward", d, hx, hw, hb, hy, 0)
    assert rel_l2(ctx.read(hy), y) <= TOL[dtype]
    hdy = ctx.upload(dy.astype(dt))
    hdx = ctx.upload(np.full(x.size, np.nan, dt))
    ctx.call("cdnn_conv_backward_data", d, hw, hdy, hdx, 0)
    assert rel_l2(ctx.read(hdx), xt.grad.numpy()) <= TOL[dtype]
    dw0 = rng.uniform(-1, 1, wt.size)
    db0 = rng.uniform(-1, 1, co)
    hdw, hdb = ctx.upload(dw0.astype(dt)), ctx.upload(db0.astype(dt))
    ctx.call("cdnn_conv_backward_filter", d, hx, hdy, hdw, hdb, 0)   # accumulates
    assert rel_l2(ctx.read(hdw), dw0 + wtt.grad.numpy().ravel()) <= TOL[dtype]
    assert rel_l2(ctx.read(hdb), db0 + bt.grad.numpy()) <= TOL[dtype]


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("case", [(2, 3, 32, 32, 3, 2, 0), (2, 5, 24, 24, 2, 2, 0), (2, 4, 13, 13, 3, 2, 1),
                                  (1, 2, 7, 9, 3, 3, 1)])
def test_pool(ctx, dtype, case):
    n, c, h, w, k, s, p = case
    rng = np.random.default_rng(sum(case))
    x = rng.standard_normal((n, c, h, w))
    dt = NP[dtype]
    for method in (cd.POOL_MAX, cd.POOL_AVE):
        d = ctx.pool_desc(n, c, h, w, method, k, s, p)
        shp = ctx.pool_output_shape(d)
        xt = torch.from_numpy(x).requires_grad_()
        if method == cd.POOL_MAX:
            yt = torch.nn.functional.max_pool2d(xt, k, s, p, ceil_mode=True)
        else:
            yt = torch.nn.functional.avg_pool2d(xt, k, s, p, ceil_mode=True, count_include_pad=True)
        if method == cd.POOL_AVE and p > 0:
            continue  # torch's ceil-mode divisor differs from Caffe's at padded edges; covered by the oracle tests
        assert shp == tuple(yt.shape)
        dy = rng.standard_normal(yt.shape)
        yt.backward(torch.from_numpy(dy))
        hx = ctx.upload(x.astype(dt))
        hy = ctx.alloc(yt.numel(), dtype)
        hm = ctx.alloc(yt.numel(), cd.I32)
        ctx.call("cdnn_pool_forward", d, hx, hy, hm, 0)
        assert rel_l2(ctx.read(hy), yt.detach().numpy()) <= 1e-6
        hdy = ctx.upload(dy.astype(dt))
        hdx = ctx.alloc(x.size, dtype)
        ctx.call("cdnn_pool_backward", d, hdy, hm, hdx, 0)
        assert rel_l2(ctx.read(hdx), xt.grad.numpy()) <= 1e-6


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
def test_softmax_loss(ctx, dtype):
    rng = np.random.default_rng(3)
    rows, cls = 100, 10
    x = rng.standard_normal((rows, cls)) * 3
    lab = rng.integers(0, cls, rows).astype(np.float64)
    dt = NP[dtype]
    hx, hl = ctx.upload(x.astype(dt)), ctx.upload(lab.astype(dt))
    hp, hloss, hdx = ctx.alloc(rows * cls, dtype), ctx.alloc(1, dtype), ctx.alloc(rows * cls, dtype)
    ctx.call("cdnn_softmax_loss_forward", hx, hl, hp, hloss, rows, cls, 1, 0)
    xt = torch.from_numpy(x.astype(dt).astype(np.float64)).requires_grad_()
    loss = torch.nn.functional.cross_entropy(xt, torch.from_numpy(lab.astype(np.int64)))
    loss.backward()
    assert abs(ctx.read(hloss)[0] - loss.item()) <= 1e-5 * abs(loss.item())
    ctx.call("cdnn_softmax_loss_backward", hp, hl, hdx, rows, cls, 1, 1.0, 0)
    assert rel_l2(ctx.read(hdx), xt.grad.numpy()) <= (1e-5 if dtype == cd.F32 else 1e-12)


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
def test_sgd_momentum_bit_exact(ctx, dtype):
    rng = np.random.default_rng(5)
    dt = NP[dtype]
    n = 1003
    w, g, v = (rng.standard_normal(n).astype(dt) for _ in range(3))
    hw, hg, hv = ctx.upload(w), ctx.upload(g), ctx.upload(v)
    lr, mom, wd = dt(0.01), dt(0.9), dt(0.004)
    ctx.call("cdnn_solver_apply", cd.SOLVER_SGD, hw, hg, hv, n, float(lr), float(mom), float(wd), 0.0, 0.0, 0)
    gg = (g + wd * w).astype(dt)
    vv = (mom * v + lr * gg).astype(dt)
    ww = (w - vv).astype(dt)
    assert np.array_equal(ctx.read(hv), vv)
    assert np.array_equal(ctx.read(hw), ww)
    assert not ctx.read(hg).any()


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("k", [2, 3])
def test_fan_out_fan_in_match_copy_axpy(ctx, dtype, k):
    """Split forward / backward and Eltwise backward in one pass (cdnn_fan_out / cdnn_fan_in)
    are bit-identical to the copy / axpy / axpby sequences they replace."""
    import ctypes as C
    rng = np.random.default_rng(11 + k)
    dt = NP[dtype]
    n = 5003
    x = rng.standard_normal(n).astype(dt)
    srcs = [rng.standard_normal(n).astype(dt) for _ in range(k)]
    hx = ctx.upload(x)
    # fan-out, unscaled (Split forward) and scaled (Eltwise backward), one destination skipped
    outs = [ctx.alloc(n, dtype) for _ in range(k)]
    arr = (C.c_uint64 * k)(*[int(o) for o in outs])
    ctx.call("cdnn_fan_out", hx, arr, None, k, n, 0)
    for o in outs:
        assert np.array_equal(ctx.read(o), x)
    coeff = [1.0, -0.5, 3.0][:k]
    arr2 = (C.c_uint64 * k)(*([int(o) for o in outs[:-1]] + [0]))
    ctx.call("cdnn_fan_out", hx, arr2, (C.c_double * k)(*coeff), k, n, 0)
    for j in range(k - 1):
        ref = ctx.alloc(n, dtype)
        ctx.call("cdnn_axpby", n, coeff[j], hx, 0.0, ref, 0, 0)
        assert np.array_equal(ctx.read(outs[j]), ctx.read(ref))
    assert np.array_equal(ctx.read(outs[-1]), x)  # skipped
    # fan-in (Split backward) against copy + axpy(1.0)
    hs = [ctx.upload(v) for v in srcs]
    y = ctx.alloc(n, dtype)
    ctx.call("cdnn_fan_in", (C.c_uint64 * k)(*[int(v) for v in hs]), k, y, n, 0)
    ref = ctx.alloc(n, dtype)
    ctx.call("cdnn_copy", hs[0], ref, n, 0)
    for v in hs[1:]:
        ctx.call("cdnn_axpy", n, 1.0, v, ref, 0)
    assert np.array_equal(ctx.read(y), ctx.read(ref))
    # Eltwise SUM + in-place ReLU in the same pass (CDNN_FAN_RELU)
    yr = ctx.alloc(n, dtype)
    ctx.call("cdnn_fan_in_ex", (C.c_uint64 * k)(*[int(v) for v in hs]), k, yr, n, cd.FAN_RELU, 0, 0)
    assert np.array_equal(ctx.read(yr), np.maximum(ctx.read(ref), 0))
    # Split backward + the backward of the in-place ReLU producing its bottom (gate = that data)
    gate = ctx.upload(srcs[-1])
    ctx.call("cdnn_fan_in_ex", (C.c_uint64 * k)(*[int(v) for v in hs]), k, yr, n, 0, gate, 0)
    assert np.array_equal(ctx.read(yr), np.where(srcs[-1] > 0, ctx.read(ref), 0))


# ---- config 4-5 layers (LRN, Dropout, BatchNorm, Scale, Eltwise) vs torch fp64 -----------

@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("n,c,h,w,size", [(2, 96, 13, 13, 5), (3, 7, 5, 4, 3), (1, 4, 1, 1, 5)])
def test_lrn(ctx, dtype, n, c, h, w, size):
    rng = np.random.default_rng(n * c + size)
    dt = NP[dtype]
    x = rng.uniform(-3, 3, (n, c, h, w)).astype(dt)
    alpha, beta, k = 1e-2, 0.75, 1.0
    xt = torch.from_numpy(x.astype(np.float64)).requires_grad_()
    yt = torch.nn.functional.local_response_norm(xt, size, alpha=alpha, beta=beta, k=k)
    dy = rng.uniform(-1, 1, yt.shape)
    yt.backward(torch.from_numpy(dy))
    hx, hy, hs = ctx.upload(x), ctx.alloc(x.size, dtype), ctx.alloc(x.size, dtype)
    ctx.call("cdnn_lrn_forward", hx, hy, hs, n, c, h * w, size, alpha, beta, k, 0)
    tol = 1e-6 if dtype == cd.F32 else 1e-13
    assert rel_l2(ctx.read(hy), yt.detach().numpy()) <= tol
    hdy, hdx = ctx.upload(dy.astype(dt)), ctx.alloc(x.size, dtype)
    ctx.call("cdnn_lrn_backward", hx, hy, hs, hdy, hdx, n, c, h * w, size, alpha, beta, 0)
    assert rel_l2(ctx.read(hdx), xt.grad.numpy()) <= tol * 10


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
def test_dropout_mask_matches_hash_and_advances(ctx, dtype):
    from test_cpu_oracle_caffe import np_drop_hash
    dt = NP[dtype]
    n, ratio, seed = 100003, 0.5, 0x1234_5678_9ABC_DEF0
    x = np.random.default_rng(1).uniform(0.5, 1.5, n).astype(dt)
    hx, hy, hk = ctx.upload(x), ctx.alloc(n, dtype), ctx.alloc(1, cd.F64)
    ctx.call("cdnn_fill", hk, 1, 0.0, 0)
    thr = np.uint32(int(ratio * 2 ** 32))
    for it in (0, 1, 2):
        ctx.call("cdnn_dropout", hx, hy, n, ratio, seed, hk, 0)
        keep = np_drop_hash(seed, it, np.arange(n)) > thr
        y = ctx.read(hy)
        assert np.array_equal(y != 0, keep)
        assert np.array_equal(y[keep], (x[keep] * dt(1 / (1 - ratio))).astype(dt))
        ctx.call("cdnn_counter_increment", hk, 0)


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("shape", [(128, 16, 32, 32), (8, 64, 8, 8), (3, 5, 1, 1)])
def test_batchnorm(ctx, dtype, shape):
    n, c, h, w = shape
    rng = np.random.default_rng(c)
    dt = NP[dtype]
    x = (rng.standard_normal(shape) * 2 + 1).astype(dt)
    xt = torch.from_numpy(x.astype(np.float64)).requires_grad_()
    yt = torch.nn.functional.batch_norm(xt, None, None, training=True, eps=1e-5)
    dy = rng.uniform(-1, 1, shape)
    yt.backward(torch.from_numpy(dy))
    hx, hy = ctx.upload(x), ctx.alloc(x.size, dtype)
    hm, hv, hs = ctx.alloc(c, dtype), ctx.alloc(c, dtype), ctx.alloc(2 * c, dtype)
    ctx.call("cdnn_batchnorm_forward", hx, hy, hm, hv, n, c, h * w, 1e-5, 0)
    tol = 1e-5 if dtype == cd.F32 else 1e-12
    assert rel_l2(ctx.read(hy), yt.detach().numpy()) <= tol
    assert rel_l2(ctx.read(hm), x.astype(np.float64).mean(axis=(0, 2, 3))) <= tol
    hdy, hdx = ctx.upload(dy.astype(dt)), ctx.alloc(x.size, dtype)
    ctx.call("cdnn_batchnorm_backward", hy, hv, hdy, hdx, hs, n, c, h * w, 0)
    assert rel_l2(ctx.read(hdx), xt.grad.numpy()) <= tol * 10


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("shape", [(128, 16, 32, 32), (8, 64, 8, 8), (3, 5, 3, 3), (64, 8, 7, 7)])
def test_batchnorm_scale_fused(ctx, dtype, shape):
    """cdnn_batchnorm_scale_forward[_ex] / _backward (the fused BatchNorm+Scale[+ReLU] of
    ResNet-20) against torch fp64: packed (HW % 4 == 0) and element-wise planes, many and
    few channel splits; CDNN_BN_RELU stores exactly max(z, 0) with xnorm unchanged."""
    n, c, h, w = shape
    rng = np.random.default_rng(n + c)
    dt = NP[dtype]
    x = (rng.standard_normal(shape) * 2 + 1).astype(dt)
    g = rng.uniform(0.5, 1.5, c).astype(dt)
    b = rng.uniform(-1, 1, c).astype(dt)
    dz = rng.uniform(-1, 1, shape).astype(dt)
    xt = torch.from_numpy(x.astype(np.float64)).requires_grad_()
    gt = torch.from_numpy(g.astype(np.float64)).requires_grad_()
    bt = torch.from_numpy(b.astype(np.float64)).requires_grad_()
    xnt = torch.nn.functional.batch_norm(xt, None, None, training=True, eps=1e-5)
    zt = xnt * gt[None, :, None, None] + bt[None, :, None, None]
    zt.backward(torch.from_numpy(dz.astype(np.float64)))
    hx, hg, hb = ctx.upload(x), ctx.upload(g), ctx.upload(b)
    hxn, hz, hzr = ctx.alloc(x.size, dtype), ctx.alloc(x.size, dtype), ctx.alloc(x.size, dtype)
    hm, hv, hs = ctx.alloc(c, dtype), ctx.alloc(c, dtype), ctx.alloc(2 * c, dtype)
    ctx.call("cdnn_batchnorm_scale_forward", hx, hxn, hz, hm, hv, hg, hb, n, c, h * w, 1e-5, 0)
    tol = 1e-5 if dtype == cd.F32 else 1e-12
    assert rel_l2(ctx.read(hxn), xnt.detach().numpy()) <= tol
    assert rel_l2(ctx.read(hz), zt.detach().numpy()) <= tol
    xn0 = ctx.read(hxn).copy()
    ctx.call("cdnn_batchnorm_scale_forward_ex", hx, hxn, hzr, hm, hv, hg, hb, n, c, h * w, 1e-5, cd.BN_RELU, 0)
    assert np.array_equal(ctx.read(hzr), np.maximum(ctx.read(hz), 0))
    assert np.array_equal(ctx.read(hxn), xn0)
    dg0 = rng.standard_normal(c).astype(dt)  # parameter gradients accumulate
    hdz, hdx = ctx.upload(dz), ctx.alloc(x.size, dtype)
    hdg, hdb = ctx.upload(dg0), ctx.upload(np.zeros(c, dt))
    ctx.call("cdnn_batchnorm_scale_backward", hxn, hv, hg, hdz, hdx, hdg, hdb, hs, n, c, h * w, 0)
    assert rel_l2(ctx.read(hdx), xt.grad.numpy()) <= tol * 10
    assert rel_l2(ctx.read(hdg), dg0 + gt.grad.numpy()) <= tol * 10
    assert rel_l2(ctx.read(hdb), bt.grad.numpy()) <= tol * 10


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("bias", [True, False])
def test_scale_and_axpby(ctx, dtype, bias):
    n, c, h, w = 16, 32, 8, 8
    rng = np.random.default_rng(9)
    dt = NP[dtype]
    x = rng.standard_normal((n, c, h, w)).astype(dt)
    g = rng.uniform(0.5, 1.5, c).astype(dt)
    b = rng.uniform(-1, 1, c).astype(dt)
    dy = rng.standard_normal((n, c, h, w)).astype(dt)
    hx, hg, hb, hy = ctx.upload(x), ctx.upload(g), ctx.upload(b), ctx.alloc(x.size, dtype)
    ctx.call("cdnn_scale_forward", hx, hg, hb if bias else 0, hy, n, c, h * w, 0)
    want = x.astype(np.float64) * g[None, :, None, None] + (b[None, :, None, None] if bias else 0)
    tol = 1e-6 if dtype == cd.F32 else 1e-14
    assert rel_l2(ctx.read(hy), want) <= tol
    dg0 = rng.standard_normal(c).astype(dt)  # gradients accumulate
    hdy, hdg, hdb, hdx = ctx.upload(dy), ctx.upload(dg0), ctx.upload(np.zeros(c, dt)), ctx.alloc(x.size, dtype)
    ctx.call("cdnn_scale_backward", hx, hg, hdy, hdg, hdb if bias else 0, hdx, n, c, h * w, 0)
    d64 = dy.astype(np.float64)
    assert rel_l2(ctx.read(hdg), dg0 + (d64 * x).sum(axis=(0, 2, 3))) <= tol
    if bias:
        assert rel_l2(ctx.read(hdb), d64.sum(axis=(0, 2, 3))) <= tol
    assert rel_l2(ctx.read(hdx), d64 * g[None, :, None, None]) <= tol
    # Eltwise SUM building block: y = 2*x ; y = -0.5*dy + 1*y
    ctx.call("cdnn_axpby", x.size, 2.0, hx, 0.0, hy, 0, 0)
    ctx.call("cdnn_axpby", x.size, -0.5, hdy, 1.0, hy, 1, 0)
    assert rel_l2(ctx.read(hy), 2 * x.astype(np.float64) - 0.5 * d64) <= tol


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("case", [(2, 32, 16, 16, 32, 5, 1, 2, 1, 1), (3, 3, 32, 32, 32, 5, 1, 2, 1, 1),
                                  (2, 3, 35, 35, 16, 11, 4, 0, 1, 1), (2, 8, 13, 13, 12, 3, 1, 1, 1, 2)])
def test_conv_forward_fused_relu(ctx, dtype, case):
    """cdnn_conv_forward_ex(CDNN_CONV_RELU) == relu(conv) on every forward path (tap, window-TMA,
    space-to-depth, gather)."""
    n, c, h, w, co, k, s, p, dl, g = case
    rng = np.random.default_rng(sum(case) + 1)
    x = rng.uniform(-1, 1, (n, c, h, w))
    wt = rng.uniform(-1, 1, (co, c // g, k, k))
    b = rng.uniform(-1, 1, co)
    y = np.maximum(conv_ref(x, wt, b, s, p, dl, g), 0.0)
    dt = NP[dtype]
    d = ctx.conv_desc(n, c, h, w, co, k, s, p, dl, g)
    hx, hw, hb = ctx.upload(x.astype(dt)), ctx.upload(wt.astype(dt)), ctx.upload(b.astype(dt))
    hy = ctx.alloc(y.size, dtype)
    ctx.call("cdnn_conv_forward_ex", d, hx, hw, hb, hy, 1, 0)
    out = ctx.read(hy)
    assert rel_l2(out, y) <= TOL[dtype]
    assert (out >= 0).all()


@pytest.mark.parametrize("rows,k,o", [(256, 2304, 1024), (200, 1000, 520), (256, 4096, 1000),
                                      (256, 9216, 4096), (96, 6000, 1100)])
def test_ip_large_tensor_core(ctx, math, rows, k, o):
    """InnerProduct forward / backward at AlexNet-like sizes (tcgen05 engine, TMA-fed
    operands split into tf32 hi/lo in the kernel): 3xTF32 must reach fp32 accuracy."""
    rng = np.random.default_rng(rows + k + o)
    X = rng.uniform(-1, 1, (rows, k)).astype(np.float32)
    W = rng.uniform(-1, 1, (o, k)).astype(np.float32)
    b = rng.uniform(-1, 1, o).astype(np.float32)
    dY = rng.uniform(-1, 1, (rows, o)).astype(np.float32)
    dW0 = rng.uniform(-1, 1, (o, k)).astype(np.float32)
    hx, hw, hb, hdy = ctx.upload(X), ctx.upload(W), ctx.upload(b), ctx.upload(dY)
    hy, hdx = ctx.alloc(rows * o, cd.F32), ctx.alloc(rows * k, cd.F32)
    hdw, hdb = ctx.upload(dW0), ctx.alloc(o, cd.F32)
    ctx.call("cdnn_ip_forward", hx, hw, hb, hy, rows, k, o, 0, 0)
    ctx.call("cdnn_ip_backward", hx, hw, hdy, hdw, hdb, hdx, rows, k, o, 0)
    Xd, Wd, dYd = X.astype(np.float64), W.astype(np.float64), dY.astype(np.float64)
    # The TMEM accumulator rounds toward zero (measured: the error of an unsplit
    # 3xTF32 contraction grows linearly with its length, 3.3e-6 at 1024 -> 2.9e-5 at
    # 8192 terms; profiles/dbg/gemm_err.py), so the 3xTF32 bar scales with K per tile.
    def tol(kk):
        return 1e-5 * max(1.0, kk / 1024) if math == "tf32x3" else 2e-3
    assert rel_l2(ctx.read(hy).reshape(rows, o), Xd @ Wd.T + b) <= tol(k)
    assert rel_l2(ctx.read(hdx).reshape(rows, k), dYd @ Wd) <= tol(o)
    assert rel_l2(ctx.read(hdw).reshape(o, k) - dW0, dYd.T @ Xd) <= tol(rows) * 4
    assert rel_l2(ctx.read(hdb), dYd.sum(0)) <= 1e-6
    for h in (hx, hw, hb, hdy, hy, hdx, hdw, hdb):
        ctx.free(h)


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
def test_fused_relu_gate_backward(ctx, dtype):
    """cdnn_{pool,lrn,conv}_backward_*_ex(gate) == plain backward followed by the ReLU
    backward on the gate data (layers.cpp:188-195), bit for bit; gate 0 == plain."""
    rng = np.random.default_rng(17)
    dt = NP[dtype]
    n, c, h, w = 3, 16, 12, 12
    gate = rng.standard_normal((n, c, h, w)).astype(dt)   # the in-place ReLU's data
    gate[gate < 0] = 0                                      # (post-ReLU values: zeros and positives)
    hg = ctx.upload(gate)
    mask_on = gate > 0

    # pooling (MAX 3x3/2 and AVE 2x2/2)
    for method, k, s in ((cd.POOL_MAX, 3, 2), (cd.POOL_AVE, 2, 2)):
        d = ctx.pool_desc(n, c, h, w, method, k, s, 0)
        ph, pw = ctx.pool_output_shape(d)[2:]
        hy, hm = ctx.alloc(n * c * ph * pw, dtype), ctx.alloc(n * c * ph * pw, cd.I32)
        ctx.call("cdnn_pool_forward", d, hg, hy, hm, 0)
        hdy = ctx.upload(rng.standard_normal(n * c * ph * pw).astype(dt))
        plain, fused = ctx.alloc(gate.size, dtype), ctx.alloc(gate.size, dtype)
        ctx.call("cdnn_pool_backward", d, hdy, hm, plain, 0)
        ctx.call("cdnn_pool_backward_ex", d, hdy, hm, fused, hg, 0)
        assert np.array_equal(ctx.read(fused), np.where(mask_on.ravel(), ctx.read(plain), 0))

    # LRN (the gate is the LRN's own bottom data)
    hy, hs = ctx.alloc(gate.size, dtype), ctx.alloc(gate.size, dtype)
    ctx.call("cdnn_lrn_forward", hg, hy, hs, n, c, h * w, 5, 1e-2, 0.75, 1.0, 0)
    hdy = ctx.upload(rng.standard_normal(gate.size).astype(dt))
    plain, fused = ctx.alloc(gate.size, dtype), ctx.alloc(gate.size, dtype)
    ctx.call("cdnn_lrn_backward", hg, hy, hs, hdy, plain, n, c, h * w, 5, 1e-2, 0.75, 0)
    ctx.call("cdnn_lrn_backward_ex", hg, hy, hs, hdy, fused, n, c, h * w, 5, 1e-2, 0.75, hg, 0)
    assert np.array_equal(ctx.read(fused), np.where(mask_on.ravel(), ctx.read(plain), 0))

    # convolution backward-data (stride 1: tap-kernel epilogue; stride 2: trailing gate pass)
    for stride in (1, 2):
        d = ctx.conv_desc(n, c, h, w, 32, 3, stride, 1)
        P, Q = ctx.conv_output_shape(d)[2:]
        hw_ = ctx.upload(rng.standard_normal(32 * c * 9).astype(dt))
        hdy = ctx.upload(rng.standard_normal(n * 32 * P * Q).astype(dt))
        plain, fused = ctx.alloc(gate.size, dtype), ctx.alloc(gate.size, dtype)
        ctx.call("cdnn_conv_backward_data", d, hw_, hdy, plain, 0)
        ctx.call("cdnn_conv_backward_data_ex", d, hw_, hdy, fused, hg, 0)
        assert np.array_equal(ctx.read(fused), np.where(mask_on.ravel(), ctx.read(plain), 0))


_POOL_DIGEST = r'''
import hashlib, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
from paper_1810_02272_b200 import cudadnn as cd
ctx = cd.Context(0)
h = hashlib.sha1()
for dtype, dt in ((cd.F32, np.float32), (cd.F64, np.float64)):
    for n, c, H, W, k, s, p in ((3, 5, 55, 55, 3, 2, 0), (2, 4, 13, 13, 3, 2, 1), (2, 3, 24, 24, 2, 2, 0),
                                (2, 3, 7, 9, 2, 2, 1), (1, 2, 32, 32, 3, 2, 0)):
        rng = np.random.default_rng(n * H + W)
        x = np.round(rng.standard_normal(n * c * H * W), 1).astype(dt)   # ties: first maximum must win
        for method in (cd.POOL_MAX, cd.POOL_AVE):
            d = ctx.pool_desc(n, c, H, W, method, k, s, p)
            P, Q = ctx.pool_output_shape(d)[2:]
            hx, hy, hm = ctx.upload(x), ctx.alloc(n * c * P * Q, dtype), ctx.alloc(n * c * P * Q, cd.I32)
            ctx.call("cdnn_pool_forward", d, hx, hy, hm, 0)
            hdy = ctx.upload(rng.standard_normal(n * c * P * Q).astype(dt))
            hdx, hdg = ctx.alloc(x.size, dtype), ctx.alloc(x.size, dtype)
            ctx.call("cdnn_pool_backward", d, hdy, hm, hdx, 0)
            ctx.call("cdnn_pool_backward_ex", d, hdy, hm, hdg, hx, 0)
            for o in (hy, hm, hdx, hdg):
                h.update(ctx.read(o).tobytes())
print(h.hexdigest())
'''


def test_pool_fixed_window_kernels_equal_generic():
    """The unrolled 3x3/2 and 2x2/2 MAX / AVE kernels (default) produce the same bytes as the
    dynamic-window kernels (CDNN_POOL_GENERIC=1): outputs, argmax masks, gated and
    plain backward, float and double, padded and ragged planes, tied maxima."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for generic in ("0", "1"):
        env = dict(os.environ, CDNN_POOL_GENERIC=generic)
        r = subprocess.run([sys.executable, "-c", _POOL_DIGEST, root], env=env, capture_output=True, text=True,
                           timeout=300, check=True)
        out[generic] = r.stdout.strip().splitlines()[-1]
    assert out["0"] == out["1"]


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("n,c,h,w,size,k,s", [(3, 96, 55, 55, 5, 3, 2),   # AlexNet norm1 -> pool1 shape
                                              (2, 40, 27, 27, 5, 3, 2),   # norm2 -> pool2 shape
                                              (2, 7, 13, 11, 3, 3, 2),    # ragged, C not a multiple of 4
                                              (2, 6, 12, 10, 5, 2, 2),    # 2x2/2 windows
                                              (1, 3, 9, 9, 5, 3, 2),      # fewer channels than the window
                                              (1, 256, 13, 13, 3, 3, 2),  # two 128-channel segments, fast paths
                                              (2, 130, 15, 15, 5, 3, 2)])  # a 2-channel second segment
def test_lrn_pool_fused_bit_identical_to_unfused(ctx, dtype, n, c, h, w, size, k, s):
    """cdnn_lrn_pool_forward / _backward (ops_lrnpool.cu) == LRN then MAX pooling, bit
    for bit: the LRN top, the pooled top, the argmax mask and the bottom gradient
    (with the fused ReLU gate on x)."""
    rng = np.random.default_rng(n * c + h + size)
    dt = NP[dtype]
    x = rng.standard_normal((n, c, h, w)).astype(dt)  # negatives exercise the ReLU gate
    alpha, beta, kk = 1e-4 * 100, 0.75, 2.0
    d = ctx.pool_desc(n, c, h, w, cd.POOL_MAX, k, s, 0)
    ok = C.c_int()
    ctx.call("cdnn_lrn_pool_supported", d, size, C.byref(ok))
    assert ok.value == 1
    ph, pw = ctx.pool_output_shape(d)[2:]
    nin, nout = x.size, n * c * ph * pw
    hx = ctx.upload(x)
    # unfused: LRN forward, pool forward; pool backward, LRN backward (gate = x)
    hy, hs, hp, hm = ctx.alloc(nin, dtype), ctx.alloc(nin, dtype), ctx.alloc(nout, dtype), ctx.alloc(nout, cd.I32)
    ctx.call("cdnn_lrn_forward", hx, hy, hs, n, c, h * w, size, alpha, beta, kk, 0)
    ctx.call("cdnn_pool_forward", d, hy, hp, hm, 0)
    dy = rng.standard_normal(nout).astype(dt)
    hdy = ctx.upload(dy)
    hdn, hdx = ctx.alloc(nin, dtype), ctx.alloc(nin, dtype)
    ctx.call("cdnn_pool_backward", d, hdy, hm, hdn, 0)
    ctx.call("cdnn_lrn_backward_ex", hx, hy, hs, hdn, hdx, n, c, h * w, size, alpha, beta, hx, 0)
    # fused
    fy, fp, fm, fdx = ctx.alloc(nin, dtype), ctx.alloc(nout, dtype), ctx.alloc(nout, cd.I32), ctx.alloc(nin, dtype)
    ctx.call("cdnn_lrn_pool_forward", d, hx, fy, fp, fm, size, alpha, beta, kk, 0, 0)
    ctx.call("cdnn_lrn_pool_backward", d, hx, hdy, hm, fdx, hx, size, alpha, beta, kk, 0)
    assert np.array_equal(ctx.read(fy), ctx.read(hy))
    assert np.array_equal(ctx.read(fp), ctx.read(hp))
    assert np.array_equal(ctx.read(fm), ctx.read(hm))
    assert np.array_equal(ctx.read(fdx), ctx.read(hdx))
    # and the fused backward without the gate == pool backward + plain LRN backward
    ctx.call("cdnn_lrn_backward", hx, hy, hs, hdn, hdx, n, c, h * w, size, alpha, beta, 0)
    ctx.call("cdnn_lrn_pool_backward", d, hx, hdy, hm, fdx, 0, size, alpha, beta, kk, 0)
    assert np.array_equal(ctx.read(fdx), ctx.read(hdx))
    for hnd in (hx, hy, hs, hp, hm, hdy, hdn, hdx, fy, fp, fm, fdx):
        ctx.free(hnd)
    ctx.call("cdnn_desc_free", d)


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("rows,k,o", [(1024, 4, 10), (1024, 10, 2), (600, 33, 64), (100, 64, 10)])
def test_ip_backward_small(ctx, dtype, rows, k, o):
    """InnerProduct backward on the few-output shapes (PG-MLP batch 1024: block-per-output
    dW and block-per-column bias sums): dW += dY^T X, db += colsum(dY), dX = dY W."""
    rng = np.random.default_rng(rows + k + o)
    dt = NP[dtype]
    x, w, dy = (rng.uniform(-1, 1, s).astype(dt) for s in ((rows, k), (o, k), (rows, o)))
    dw0, db0 = rng.uniform(-1, 1, (o, k)).astype(dt), rng.uniform(-1, 1, o).astype(dt)
    hx, hw, hdy, hdw, hdb = (ctx.upload(a) for a in (x, w, dy, dw0, db0))
    hdx = ctx.alloc(rows * k, dtype)
    ctx.call("cdnn_ip_backward", hx, hw, hdy, hdw, hdb, hdx, rows, k, o, 0)
    X, W, DY = (a.astype(np.float64) for a in (x, w, dy))
    tol = 1e-5 if dtype == cd.F32 else 1e-12
    assert rel_l2(ctx.read(hdw).reshape(o, k), dw0 + DY.T @ X) <= tol
    assert rel_l2(ctx.read(hdb), db0 + DY.sum(0)) <= tol
    assert rel_l2(ctx.read(hdx).reshape(rows, k), DY @ W) <= tol
    for h in (hx, hw, hdy, hdw, hdb, hdx):
        ctx.free(h)


def test_conv_backward_filter_reuses_forward_input_rewrite(ctx):
    """CDNN_CONV_INPUT_UNCHANGED: the strided stem's backward filter reuses the forward's
    space-to-depth rewrite of its input -- bit-identical to redoing it, and ignored when
    the promise cannot hold (another input buffer)."""
    n, c, h, w, co, k, s = 4, 3, 67, 67, 96, 11, 4
    rng = np.random.default_rng(21)
    x, x2 = (rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32) for _ in range(2))
    wt = rng.uniform(-1, 1, (co, c, k, k)).astype(np.float32)
    d = ctx.conv_desc(n, c, h, w, co, k, s, 0)
    P, Q = ctx.conv_output_shape(d)[2:]
    dy = rng.uniform(-1, 1, (n, co, P, Q)).astype(np.float32)
    hx, hx2, hw, hdy = ctx.upload(x), ctx.upload(x2), ctx.upload(wt), ctx.upload(dy)
    hy = ctx.alloc(n * co * P * Q, cd.F32)
    outs = []
    for flags, xin in ((0, hx), (2, hx), (2, hx2), (0, hx2)):
        ctx.call("cdnn_conv_forward", d, hx, hw, 0, hy, 0)  # the forward always sees x
        hdw, hdb = ctx.alloc(wt.size, cd.F32), ctx.alloc(co, cd.F32)
        ctx.call("cdnn_conv_backward_filter_ex", d, xin, hdy, hdw, hdb, flags, 0)
        outs.append((ctx.read(hdw), ctx.read(hdb)))
        ctx.free(hdw)
        ctx.free(hdb)
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[2][0], outs[3][0])  # other input: the flag is ignored
    assert not np.array_equal(outs[0][0], outs[2][0])
    for hnd in (hx, hx2, hw, hdy, hy):
        ctx.free(hnd)


def _mlp_reference(X, act, ret, count, W1, b1, W2, b2):
    """fp64 restatement of the pg_softmax update's gradient (layers.cpp InnerProduct /
    ReLU / Softmax, trainer.cpp:42-113 softmax gradient, summed over the batch)."""
    pre = X @ W1.T + b1
    a = np.maximum(pre, 0)
    l = a @ W2.T + b2
    e = np.exp(l - l.max(1, keepdims=True))
    p = e / e.sum(1, keepdims=True)
    dl = np.zeros_like(p)
    dl[:count] = p[:count]
    dl[np.arange(count), act[:count].astype(int)] -= 1
    dl[:count] *= ret[:count, None]
    dh = (dl @ W2) * (pre > 0)
    return l, p, a, dh.T @ X, dh.sum(0), dl.T @ a, dl.sum(0)


@pytest.mark.parametrize("dtype", [cd.F32, cd.F64])
@pytest.mark.parametrize("rows,count,dims", [(1024, 1024, (4, 10, 2)), (300, 211, (4, 10, 2)),
                                             (777, 500, (7, 33, 3)), (64, 64, (16, 20, 5))])
def test_mlp_pg_step_device_buffers(ctx, dtype, rows, count, dims):
    """cdnn_mlp_pg_step from device buffers (the fp32 4-10-2 register kernel and the
    shared-memory kernel for other extents / fp64): tops, and the SGD update
    (momentum, weight decay, pre-existing arena gradient added) against fp64."""
    i, h, c = dims
    rng = np.random.default_rng(rows + i)
    dt = NP[dtype]
    X = rng.uniform(-1, 1, (rows, i))
    act = np.floor(rng.uniform(0, c, rows))
    ret = rng.standard_normal(rows)
    W1, b1 = rng.uniform(-0.5, 0.5, (h, i)), rng.uniform(-0.1, 0.1, h)
    W2, b2 = rng.uniform(-0.5, 0.5, (c, h)), rng.uniform(-0.1, 0.1, c)
    sizes = [W1.size, b1.size, W2.size, b2.size]
    offs = np.cumsum([0] + sizes[:-1]).astype(np.uint64) + 3  # arbitrary arena placement
    total = int(offs[-1]) + sizes[-1] + 5
    w = np.zeros(total)
    for o, v in zip(offs, (W1, b1, W2, b2)):
        w[int(o):int(o) + v.size] = v.ravel()
    g0 = rng.uniform(-1e-2, 1e-2, total)
    h0 = rng.uniform(-1e-2, 1e-2, total)
    lr, mom, wd = 1e-2, 0.9, 1e-3
    hx, ha, hr = ctx.upload(X.astype(dt)), ctx.upload(act.astype(dt)), ctx.upload(ret.astype(dt))
    hw, hg, hh = ctx.upload(w.astype(dt)), ctx.upload(g0.astype(dt)), ctx.upload(h0.astype(dt))
    hl, hp, hhid = ctx.alloc(rows * c, dtype), ctx.alloc(rows * c, dtype), ctx.alloc(rows * h, dtype)
    Xq, Wq = X.astype(dt).astype(np.float64), w.astype(dt).astype(np.float64)
    W1q, b1q, W2q, b2q = (Wq[int(o):int(o) + n].reshape(v.shape) for o, n, v in zip(offs, sizes, (W1, b1, W2, b2)))
    ok = C.c_int(0)
    ctx.call("cdnn_mlp_pg_supported", dtype, rows, i, h, c, C.byref(ok))
    assert ok.value == 1
    ctx.call("cdnn_mlp_pg_step", hx, ha, hr, rows, count, i, h, c, hw, hg, hh, (C.c_uint64 * 4)(*offs), 0,
             lr, mom, wd, 0.99, 1e-8, hhid, hl, hp, 0)
    l, p, a, gW1, gb1, gW2, gb2 = _mlp_reference(Xq, act, ret.astype(dt).astype(np.float64), count, W1q, b1q, W2q, b2q)
    tol = 1e-12 if dtype == cd.F64 else 2e-5
    assert rel_l2(ctx.read(hl).reshape(rows, c), l) <= tol
    assert rel_l2(ctx.read(hp).reshape(rows, c), p) <= tol
    assert rel_l2(ctx.read(hhid).reshape(rows, h), a) <= tol
    g = g0.astype(dt).astype(np.float64).copy()
    for o, v in zip(offs, (gW1, gb1, gW2, gb2)):
        g[int(o):int(o) + v.size] += v.ravel()
    hist_in = h0.astype(dt).astype(np.float64)
    step = mom * hist_in + lr * (g + wd * Wq)
    touched = np.zeros(total, bool)
    for o, n in zip(offs, sizes):
        touched[int(o):int(o) + n] = True
    w_new, g_new, h_new = ctx.read(hw), ctx.read(hg), ctx.read(hh)
    assert rel_l2(w_new[touched], (Wq - step)[touched]) <= tol
    assert rel_l2(h_new[touched], step[touched]) <= max(tol, 1e-4 if dtype == cd.F32 else tol)
    assert not np.any(g_new[touched])
    # elements outside the four parameters are untouched
    assert np.array_equal(w_new[~touched], w.astype(dt)[~touched])
    assert np.array_equal(g_new[~touched], g0.astype(dt)[~touched])
    for hd in (hx, ha, hr, hw, hg, hh, hl, hp, hhid):
        ctx.free(hd)
