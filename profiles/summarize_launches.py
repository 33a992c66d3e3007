"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) of
profiles/prof_step.py: the last `per_step` launches form one training step.
Usage: python profiles/summarize_launches.py launches.csv [per_step]"""
import csv
import re
import sys
from collections import OrderedDict


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name.replace("(anonymous namespace)::", "").replace("unnamed>::", ""))
    return name.replace("void ", "")[:110]


def main(path, per_step=None):
    rows = []
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] == "gpu__time_duration.sum":
            rows.append((short(r["Kernel Name"]), float(r["Metric Value"].replace(",", "")) / 1e3, r["Grid Size"],
                         r["Block Size"]))
    step = rows[-per_step:] if per_step else rows
    total = sum(t for _, t, _, _ in step)
    print(f"# {len(step)} launches, {total:.1f} us serialised (cold-cache, ncu --clock-control none)")
    print(f"{'us':>9} {'share':>6}  grid / block  kernel")
    for n, t, g, b in step:
        print(f"{t:9.2f} {100 * t / total:5.1f}%  {g}/{b}  {n}")
    agg = OrderedDict()
    for n, t, _, _ in step:
        agg[n] = agg.get(n, 0.0) + t
    print("\n# by kernel")
    for n, t in sorted(agg.items(), key=lambda kv: -kv[1]):
        print(f"{t:9.2f} {100 * t / total:5.1f}%  {n}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else None)
