"""Shared helpers for the parity tests: synthetic inputs, the
per-tensor error metrics and lock-step training of the
B200 net against the CPU oracle."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import pyoracle  # noqa: E402  (test infrastructure only)
from paper_1810_02272_b200 import polegrad  # noqa: E402

# Tolerances from north_star: 1e-5 relative (FP64) and 2e-3 relative (TF32)
# after 10 iterations, measured per tensor as relative L2 error.
TOL = {"f64": 1e-5, "f32": 2e-3}

CONFIGS = {
    # model, solver kwargs, classes, batch override (None = the prototxt's)
    "lenet": ("lenet", dict(method="sgd", lr=0.01, momentum=0.9, weight_decay=5e-4), 10, None),
    "cifar10_quick": ("cifar10_quick", dict(method="sgd", lr=0.001, momentum=0.9, weight_decay=4e-3), 10, None),
    "pg_mlp": ("pg_mlp", dict(method="rmsprop", lr=1e-3, rms_decay=0.99, epsilon=1e-8), 2, None),
    # AlexNet at a reduced batch: the oracle's naive GEMM needs ~2 s per image-iteration
    # (SURVEY §7 item 8); ResNet-20 at batch 16 (per-rank BN statistics over 16 images)
    "alexnet": ("alexnet", dict(method="sgd", lr=0.001, momentum=0.9, weight_decay=5e-4), 1000, 2),
    "resnet20": ("resnet20", dict(method="sgd", lr=0.1, momentum=0.9, weight_decay=1e-4), 10, 16),
}


def report(section: str, key: str, data) -> None:
    """Achieved errors, collected into $PARITY_REPORT_DIR/parity.json when set
    (committed as profiles/r02_parity.json)."""
    import json
    d = os.environ.get("PARITY_REPORT_DIR")
    if not d:
        return
    os.makedirs(d, exist_ok=True)
    path = os.path.join(d, "parity.json")
    cur = json.load(open(path)) if os.path.exists(path) else {}
    cur.setdefault(section, {})[key] = data
    with open(path, "w") as f:
        json.dump(cur, f, indent=1, default=float)


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    d = float(np.linalg.norm(a - b))
    n = float(np.linalg.norm(b))
    return d / n if n > 0 else d


def synthetic_batches(shape, classes, iters, seed=2):
    """U(-1,1) NCHW data and floor(u*C) labels, drawn from one stream."""
    rng = np.random.default_rng(seed)
    out = []
    for _ in range(iters):
        x = rng.uniform(-1.0, 1.0, shape)
        y = np.floor(rng.uniform(0.0, 1.0, shape[0]) * classes)
        out.append((x, y))
    return out


def data_shape(text: str):
    _, info = pyoracle.to_spec(text)
    return tuple(info["data"][2]), len(info["data"][1]) == 2


def feed_forward_state(text: str, net, orc) -> dict:
    """Oracle-fed backward: copy the B200 forward state (every layer top and
    the MAX-pool argmax masks) into the oracle so both backward passes start
    from identical activations and routing decisions.  Returns how many
    pooling-mask entries / ReLU gates differed before the copy (near-tie flips)."""
    flips = {"pool": 0, "relu": 0, "elements": 0, "top_rel": {}}
    for name, ltype, tops in pyoracle.layer_tops(text):
        if ltype in ("MemoryData", "SoftmaxWithLoss", "MemoryLoss"):
            continue
        for top in tops:
            mine = net.blob(top).astype(np.float64)
            theirs = orc.blob(top)
            # every layer's top against the oracle's own forward, before it is overwritten
            # (in-place layers report the blob after the last in-place writer)
            flips["top_rel"][top] = rel_l2(mine, theirs)
            if ltype == "ReLU":
                flips["relu"] += int(np.count_nonzero((mine > 0) != (theirs > 0)))
            orc.set_blob(top, mine)
            flips["elements"] += mine.size
        if ltype == "Pooling":
            cnt = int(np.prod(net.blob_shape(tops[0])))
            mask = net.pool_mask(name)[:cnt]
            try:
                flips["pool"] += int(np.count_nonzero(mask != orc.pool_mask(name, cnt)))
                orc.set_pool_mask(name, mask)
            except pyoracle.OracleError:
                pass  # AVE pooling keeps no mask
    return flips


# Free-running float comparisons run at a learning rate where the two float
# trajectories do not separate chaotically (profiles/r02_lr_chaos.json: at the bench
# learning rates one near-tie ReLU / max-pool flip, amplified through momentum,
# moves the zero-initialised biases of LeNet / AlexNet / ResNet-20 by 1e-2 .. 1 relative
# within ten iterations -- for the reference float build against its own float64
# build as much as for the B200).  The per-iteration gradient test on synced weights
# keeps the bench learning rates.
FREE_RUN_LR = {"lenet": 1e-3, "alexnet": 1e-4, "resnet20": 1e-3}


def per_layer(params, values):
    """Concatenate each layer's parameter tensors (name 'layer.weight' / 'layer.bias')."""
    out = {}
    for (name, _), v in zip(params, values):
        out.setdefault(name.rsplit(".", 1)[0], []).append(np.asarray(v, np.float64).ravel())
    return {k: np.concatenate(v) for k, v in out.items()}


def lockstep(config: str, dtype: str, iters: int = 10, seed: int = 1, resync_weights: bool = False,
             feed_forward: bool = False, lr: float = None):
    """Train the B200 Net and the oracle side by side from identical weights
    and inputs; returns per-iteration losses/metrics and the final nets.

    resync_weights: copy the oracle's weights into the B200 net (MCWT) before
    every iteration, so each iteration's gradients are compared on identical
    inputs AND weights.  In float, the two implementations' ~1e-7 rounding
    differences flip max-pool argmaxes / ReLU gates at near-ties; free-running
    trajectories amplify those flips in the gradients of the first layers
    (SURVEY §7.3 item 5), so gradient parity is asserted per iteration on
    synced weights, while losses and weights are asserted free-running."""
    model, skw, classes, batch = CONFIGS[config]
    if lr is not None:
        skw = dict(skw, lr=lr)
    text = polegrad.load_model(model, batch)
    shape, labelled = data_shape(text)
    net = polegrad.Net(text, seed=seed, dtype=dtype)
    orc = pyoracle.OracleNet(text, seed=seed, dtype=dtype)
    solver = polegrad.Solver(net, **skw)
    osolver = pyoracle.OracleSolver(orc, **skw)
    # same seeded init on both sides
    init_params = [orc.param(i) for i in range(len(net.param_info()))]
    init_bitexact = all(np.array_equal(net.param(i).astype(np.float64), init_params[i])
                        for i in range(len(net.param_info())))
    batches = synthetic_batches(shape, classes, iters)
    diff_rng = np.random.default_rng(3)
    hist = []
    for x, y in batches:
        if resync_weights:
            net.restore(orc.snapshot())
        if labelled:
            net.set_batch(x, y)
            orc.set_batch(x, y)
            net.forward()
            lo = orc.forward()
            l = net.loss()
            flips = feed_forward_state(text, net, orc) if feed_forward else None
            net.backward()
            orc.backward()
        else:  # PG: inject policy-gradient diffs at the logits, backward_from (trainer.cpp:171-216)
            net.set_batch(x)
            orc.set_batch(x)
            net.forward()
            orc.forward()
            g = diff_rng.uniform(-1.0, 1.0, net.blob_shape("logits"))
            net.set_blob("logits", g, diff=True)
            orc.set_blob("logits", g, diff=True)
            net.backward_from("logits")
            orc.backward_from("logits")
            l = float(np.sum(net.blob("prob")))
            lo = float(np.sum(orc.blob("prob")))
            flips = None
        grads = [rel_l2(net.param(i, diff=True), orc.param(i, diff=True)) for i in range(len(net.param_info()))]
        solver.apply()
        osolver.apply()
        hist.append({"loss": l, "oracle_loss": lo, "grad_rel": grads, "flips": flips})
    n = len(net.param_info())
    mine = [net.param(i) for i in range(n)]
    theirs = [orc.param(i) for i in range(n)]
    weights = [rel_l2(a, b) for a, b in zip(mine, theirs)]
    lm, lt = per_layer(net.param_info(), mine), per_layer(net.param_info(), theirs)
    return {"net": net, "oracle": orc, "hist": hist, "weights_rel": weights, "init_bitexact": init_bitexact,
            "params": net.param_info(), "layers_rel": {k: rel_l2(lm[k], lt[k]) for k in lm},
            "zero_init": [not np.any(init) for init in init_params]}
