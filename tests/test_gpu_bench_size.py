"""Per-layer parity of the BENCHED step at bench size.

bench.py times AlexNet at batch 256 and ResNet-20 at batch 128; the engine
behind each Convolution / InnerProduct (SIMT vs tcgen05 GEMM, split-K counts,
tap / wtap / space-to-depth / zero-insert routes) is chosen from the layer
shape, so the lock-step tests at batch 2 / 16 (test_gpu_parity.py) do not
cover the kernels that produce the headline number.  Here the full net runs
one training step (forward + backward, f32 = 3xTF32) at the bench batch, and
for every Convolution and InnerProduct layer its three products are compared
with torch float64 on the host, computed from the layer's own operands read
back from the device:

  forward  top     = conv(bottom, W) + b            (ReLU / Dropout applied when
                                                     an in-place ReLU / Dropout
                                                     rewrote the top)
  backward W.diff  = conv_weight_grad(bottom, top.diff)   b.diff = sum top.diff
  backward bottom.diff = conv_input_grad(W, top.diff)     (gated by the in-place
                                                     ReLU / Dropout that shares
                                                     the bottom blob)

Where an in-place BatchNorm / Scale rewrote the top (ResNet) or the bottom's
diff, that product is not observable in the net's blobs afterwards; it is then
checked through the same C-ABI entry point (cdnn_conv_forward /
cdnn_conv_backward_data) at exactly the layer's shape on the layer's own data.

Host cost is bounded by sampling: forward and backward-data on 8 images
(per-image independent), backward-filter on 8 output channels per group over
the whole batch, InnerProduct rows / outputs likewise.  The bar is 1e-4
relative L2 per tensor (3xTF32 reaches ~1e-6; north_star's TF32 bar is 2e-3);
the achieved errors are written to $PARITY_REPORT_DIR when set
(profiles/r02_parity_bench_size.json).
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest
import torch

from parity_util import polegrad, pyoracle, rel_l2, synthetic_batches

pytestmark = pytest.mark.gpu

TOL = 1e-4
IMGS = 8        # images sampled for forward / backward-data
OUT_CH = 8      # output channels (per group) / InnerProduct outputs sampled for backward-filter
BENCH = {"alexnet": (256, 1000), "resnet20": (128, 10)}


def _layers(text: str):
    """Layer list with parsed params (from the oracle's prototxt reader)."""
    spec, _ = pyoracle.to_spec(text)
    out = []
    for line in spec.strip().split("\n"):
        t, name, bottoms, tops, kv = line.split("|")
        p = {}
        for item in filter(None, kv.split(";")):
            k, v = item.split("=")
            p[k] = float(v)
        out.append({"type": t, "name": name, "bottoms": [b for b in bottoms.split(",") if b],
                    "tops": [b for b in tops.split(",") if b], "p": p})
    return out


def _with_split_names(layers):
    """The bottom blob names the B200 net actually wires (Caffe InsertSplits naming,
    csrc/polegrad/net.cpp with_splits): reader j of a fanned-out blob version reads
    '<blob>_<producer>_<j>_split'."""
    versions, live = [], {}
    for i, l in enumerate(layers):
        for b, name in enumerate(l["bottoms"]):
            if name in live:
                versions[live[name]]["readers"].append((i, b))
        for t in l["tops"]:
            versions.append({"name": t, "producer": i, "readers": []})
            live[t] = len(versions) - 1
    renamed = {}
    for v in versions:
        if len(v["readers"]) < 2:
            continue
        for j, (li, bi) in enumerate(v["readers"]):
            renamed[(li, bi)] = f"{v['name']}_{layers[v['producer']]['name']}_{j}_split"
    for i, l in enumerate(layers):
        l["wired"] = [renamed.get((i, b), n) for b, n in enumerate(l["bottoms"])]
    return layers


def _inplace_after(layers, i, blob):
    """Types of the in-place layers after layer i that rewrite `blob`."""
    return [l["type"] for l in layers[i + 1:] if blob in l["tops"] and blob in l["bottoms"]]


def _inplace_before(layers, i, blob):
    """Types of the in-place layers before layer i that rewrote `blob` (whose backward
    runs after layer i's and rewrites the blob's diff in place)."""
    return [l["type"] for l in layers[:i] if blob in l["tops"] and blob in l["bottoms"]]


def _dropout_scale(layers, types_and_names):
    s = 1.0
    for l in types_and_names:
        if l["type"] == "Dropout":
            s /= 1.0 - l["p"].get("dropout_ratio", 0.5)
    return s


def _conv_geom(l, cin):
    p = l["p"]
    kh, kw = int(p.get("kernel_h", 1)), int(p.get("kernel_w", 1))
    return dict(co=int(p["num_output"]), kh=kh, kw=kw, sh=int(p.get("stride_h", 1)), sw=int(p.get("stride_w", 1)),
                ph=int(p.get("pad_h", 0)), pw=int(p.get("pad_w", 0)), dil=int(p.get("dilation", 1)),
                g=int(p.get("group", 1)), cin=cin, bias=p.get("bias_term", 1.0) != 0.0)


def _t(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float64))


def _conv_fwd(x, w, b, gm):
    y = torch.nn.functional.conv2d(_t(x), _t(w), None if b is None else _t(b), stride=(gm["sh"], gm["sw"]),
                                   padding=(gm["ph"], gm["pw"]), dilation=gm["dil"], groups=gm["g"])
    return y.numpy()


def _conv_dgrad(xshape, w, dy, gm):
    return torch.nn.grad.conv2d_input(xshape, _t(w), _t(dy), stride=(gm["sh"], gm["sw"]),
                                      padding=(gm["ph"], gm["pw"]), dilation=gm["dil"], groups=gm["g"]).numpy()


def _conv_wgrad_sampled(x, dy, gm, sel_per_group):
    """dW rows for the sampled output channels, group by group, over the whole batch."""
    co, g = gm["co"], gm["g"]
    cg, og = gm["cin"] // g, co // g
    rows, idx = [], []
    for gi in range(g):
        sel = [gi * og + s for s in sel_per_group if s < og]
        xg = _t(x[:, gi * cg:(gi + 1) * cg])
        dw = torch.nn.grad.conv2d_weight(xg, (len(sel), cg, gm["kh"], gm["kw"]), _t(dy[:, sel]),
                                         stride=(gm["sh"], gm["sw"]), padding=(gm["ph"], gm["pw"]),
                                         dilation=gm["dil"])
        rows.append(dw.numpy())
        idx += sel
    return np.concatenate(rows), idx


def _report(name: str, rows: list) -> None:
    d = os.environ.get("PARITY_REPORT_DIR")
    if not d:
        return
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, "parity_bench_size.json")
    cur = json.load(open(path)) if os.path.exists(path) else {}
    cur[name] = rows
    with open(path, "w") as f:
        json.dump(cur, f, indent=1)


@pytest.mark.parametrize("model", ["alexnet", "resnet20"])
def test_bench_size_layers_match_fp64(ctx, model):
    torch.set_num_threads(max(1, min(32, os.cpu_count() or 1)))
    batch, classes = BENCH[model]
    text = polegrad.load_model(model, batch)
    layers = _with_split_names(_layers(text))
    net = polegrad.Net(text, seed=1, dtype="f32")
    shape = (batch,) + net.blob_shape("data")[1:]
    (x, y), = synthetic_batches(shape, classes, 1)
    net.set_batch(x, y)
    net.forward()
    loss = net.loss()
    net.backward()
    net.sync()
    assert np.isfinite(loss)
    params = {name: i for i, (name, _) in enumerate(net.param_info())}
    rng = np.random.default_rng(7)
    imgs = np.unique(np.concatenate([[0, batch - 1], rng.choice(batch, IMGS - 2, replace=False)]))
    rows = []
    from paper_1810_02272_b200 import cudadnn as cd

    for i, l in enumerate(layers):
        if l["type"] not in ("Convolution", "InnerProduct"):
            continue
        name, top, bottom = l["name"], l["tops"][0], l["wired"][0]
        W = net.param(params[f"{name}.weight"]).astype(np.float64)
        dW = net.param(params[f"{name}.weight"], diff=True).astype(np.float64)
        has_b = f"{name}.bias" in params
        B = net.param(params[f"{name}.bias"]).astype(np.float64).ravel() if has_b else None
        dB = net.param(params[f"{name}.bias"], diff=True).astype(np.float64).ravel() if has_b else None
        X = net.blob(bottom).astype(np.float64)
        T = net.blob(top).astype(np.float64)
        dT = net.blob(top, diff=True).astype(np.float64)
        dX = net.blob(bottom, diff=True).astype(np.float64)
        after = [l2 for l2 in layers[i + 1:] if top in l2["tops"] and top in l2["bottoms"]]
        before = [l2 for l2 in layers[:i] if bottom in l2["tops"] and bottom in l2["bottoms"]]
        top_observable = all(a["type"] in ("ReLU", "Dropout") for a in after)
        bottom_observable = all(b["type"] in ("ReLU", "Dropout") for b in before)
        propagate = bottom not in layers[0]["tops"]  # no gradient into the data blob (Caffe need-backward)
        r = {"layer": name, "type": l["type"], "bottom": bottom, "top_shape": list(T.shape)}

        if l["type"] == "InnerProduct":
            Xr = X.reshape(batch, -1)
            dTr = dT.reshape(batch, -1)
            Yf = Xr[imgs] @ W.reshape(W.shape[-2], -1).T + (B if has_b else 0.0)
            W2 = W.reshape(W.shape[-2], -1)
            sel = rng.choice(W2.shape[0], min(64, W2.shape[0]), replace=False)
            want_dw = dTr[:, sel].T @ Xr
            r["wgrad"] = rel_l2(dW.reshape(W2.shape)[sel], want_dw)
            want_dx = dTr[imgs] @ W2
            geom_conv = None
        else:
            gm = _conv_geom(l, X.shape[1])
            Yf = _conv_fwd(X[imgs], W, B, gm)
            sel_pg = list(rng.choice(gm["co"] // gm["g"], min(OUT_CH, gm["co"] // gm["g"]), replace=False))
            want_dw, idx = _conv_wgrad_sampled(X, dT, gm, sel_pg)
            r["wgrad"] = rel_l2(dW[idx], want_dw)
            want_dx = _conv_dgrad(X[imgs].shape, W, dT[imgs], gm)
            geom_conv = gm
        if has_b:
            r["bgrad"] = rel_l2(dB, dT.reshape(batch, dB.size, -1).sum(axis=(0, 2)))

        # forward
        if top_observable:
            got = T[imgs].reshape(Yf.shape)
            want = Yf
            if any(a["type"] == "ReLU" for a in after):
                want = np.maximum(want, 0.0)
            if any(a["type"] == "Dropout" for a in after):
                want = want * _dropout_scale(layers, after) * (got != 0)
            r["forward"] = rel_l2(got, want)
            r["forward_where"] = "in situ"
        else:  # rewritten in place by BatchNorm / Scale: same entry point, same shape
            gm = geom_conv
            d = ctx.conv_desc(batch, gm["cin"], X.shape[2], X.shape[3], gm["co"], (gm["kh"], gm["kw"]),
                              (gm["sh"], gm["sw"]), (gm["ph"], gm["pw"]), gm["dil"], gm["g"])
            hx, hw = ctx.upload(X.astype(np.float32)), ctx.upload(W.astype(np.float32))
            hb = ctx.upload(B.astype(np.float32)) if has_b else 0
            hy = ctx.alloc(int(np.prod(T.shape)), cd.F32)
            ctx.call("cdnn_conv_forward", d, hx, hw, hb, hy, 0)
            got = ctx.read(hy).reshape(T.shape)[imgs].astype(np.float64)
            r["forward"] = rel_l2(got, Yf)
            r["forward_where"] = "cdnn_conv_forward at the layer shape"
            for h in (hx, hw, hy) + ((hb,) if has_b else ()):
                ctx.free(h)
            ctx.call("cdnn_desc_free", d)

        # backward-data
        if propagate:
            if bottom_observable:
                got = dX[imgs].reshape(want_dx.shape)
                want = want_dx
                if before:
                    want = want * _dropout_scale(layers, before) * (X[imgs].reshape(want.shape) != 0)
                r["dgrad"] = rel_l2(got, want)
                r["dgrad_where"] = "in situ"
            else:
                gm = geom_conv
                d = ctx.conv_desc(batch, gm["cin"], X.shape[2], X.shape[3], gm["co"], (gm["kh"], gm["kw"]),
                                  (gm["sh"], gm["sw"]), (gm["ph"], gm["pw"]), gm["dil"], gm["g"])
                hw, hdy = ctx.upload(W.astype(np.float32)), ctx.upload(dT.astype(np.float32))
                hdx = ctx.alloc(X.size, cd.F32)
                ctx.call("cdnn_conv_backward_data", d, hw, hdy, hdx, 0)
                got = ctx.read(hdx).reshape(X.shape)[imgs].astype(np.float64)
                r["dgrad"] = rel_l2(got, want_dx)
                r["dgrad_where"] = "cdnn_conv_backward_data at the layer shape"
                for h in (hw, hdy, hdx):
                    ctx.free(h)
                ctx.call("cdnn_desc_free", d)
        rows.append(r)
    _report(model, rows)
    print(json.dumps(rows, indent=None))
    assert rows, "no Convolution / InnerProduct layers found"
    bad = [(r["layer"], k, r[k]) for r in rows for k in ("forward", "wgrad", "bgrad", "dgrad")
           if k in r and not r[k] <= TOL]
    assert not bad, bad
