"""Achieved parity errors of the B200 library against the CPU oracle, per config
and dtype (run on a GPU box; writes JSON): free-running 10-iteration lock-step
(loss error per iteration, per-tensor weight error after 10 updates, per-tensor
gradient error per iteration) and the synced-weight / oracle-fed gradient run.

    python profiles/parity_report.py [out.json] [config ...]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests"))
sys.path.insert(0, ROOT)

from parity_util import CONFIGS, lockstep  # noqa: E402


def summarize(r):
    names = [n for n, _ in r["params"]]
    return {
        "loss_rel": [abs(h["loss"] - h["oracle_loss"]) / max(abs(h["oracle_loss"]), 1e-12) for h in r["hist"]],
        "grad_rel_max_per_iter": [max(h["grad_rel"]) for h in r["hist"]],
        "grad_rel_worst_tensor": max(((e, n) for h in r["hist"] for n, e in zip(names, h["grad_rel"])))[1],
        "weights_rel": dict(zip(names, r["weights_rel"])),
        "weights_rel_max": max(r["weights_rel"]),
        "flips": [h["flips"] for h in r["hist"] if h.get("flips")],
    }


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else "parity_report.json"
    configs = sys.argv[2:] or list(CONFIGS)
    rep = {}
    for cfg in configs:
        for dt in ("f64", "f32"):
            key = f"{cfg}.{dt}"
            try:
                rep[key] = {"free": summarize(lockstep(cfg, dt, iters=10)),
                            "synced": summarize(lockstep(cfg, dt, iters=10, resync_weights=True, feed_forward=True))}
            except Exception as e:  # keep going: this is a report
                rep[key] = {"error": repr(e)}
            print(key, json.dumps({k: (v if k == "error" else {kk: vv for kk, vv in v.items()
                                                               if kk in ("loss_rel", "weights_rel_max")})
                                   for k, v in rep[key].items()}), flush=True)
            with open(out, "w") as f:
                json.dump(rep, f, indent=1)


if __name__ == "__main__":
    main()
