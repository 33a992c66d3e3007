"""How fast do free-running float trajectories (B200 f32 vs the reference float
build) separate, as a function of the learning rate?  Prints, per config and lr
multiplier, the worst per-iteration loss error and the worst per-tensor weight
error after 10 iterations (tooling for choosing the parity-test solver)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)
import parity_util as pu  # noqa: E402

out = {}
for cfg in sys.argv[1:] or ["lenet", "alexnet", "resnet20"]:
    base = pu.CONFIGS[cfg]
    for mult in (1.0, 0.1, 0.01):
        skw = dict(base[1])
        skw["lr"] = skw["lr"] * mult
        pu.CONFIGS[cfg] = (base[0], skw, base[2], base[3])
        r = pu.lockstep(cfg, "f32", iters=10)
        loss = [abs(h["loss"] - h["oracle_loss"]) / abs(h["oracle_loss"]) for h in r["hist"]]
        w = sorted(zip(r["weights_rel"], [n for n, _ in r["params"]]), reverse=True)[:3]
        out[f"{cfg} lr*{mult}"] = {"lr": skw["lr"], "loss_max": max(loss), "weights_worst": w}
        print(f"{cfg} lr={skw['lr']:g}: loss err max {max(loss):.3g}, worst weights {w}", flush=True)
        pu.CONFIGS[cfg] = base
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "lr_chaos.json"), "w"), indent=1)
