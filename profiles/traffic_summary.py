"""Per-launch DRAM traffic of the bench's dominant layer op (CIFAR-10 quick
conv2 backward = backward-filter tap kernel + its split reduce + weight repack
+ backward-data tap kernel) from an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
(default cache control: caches flushed before every kernel, i.e. cold).
Usage: python profiles/traffic_summary.py launches_dram_cold.csv > profiles/ncu_summary.json"""
import csv
import json
import sys
from collections import OrderedDict


def main(path):
    lines = [l for l in open(path) if l.startswith('"')]
    launches = OrderedDict()
    for r in csv.DictReader(lines):
        d = launches.setdefault(r["ID"], {"name": r["Kernel Name"]})
        d[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    L = list(launches.values())
    nbytes = lambda x: x.get("dram__bytes_read.sum", 0.0) + x.get("dram__bytes_write.sum", 0.0)
    # last occurrence of the conv2-backward group: wtap<32> -> reduce -> repack -> conv_tap
    idx = max(i for i, x in enumerate(L) if "conv_wtap_kernel<32" in x["name"])
    group = L[idx:idx + 4]
    assert "reduce_splits" in group[1]["name"] and "repack_tap" in group[2]["name"] and "conv_tap_kernel" in group[3]["name"]
    out = {
        "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (cold caches), "
                  "python profiles/prof_step.py 2, B200",
        "traffic_bytes_per_launch": {"conv2.bwd": sum(nbytes(x) for x in group)},
        "kernels": {"conv2.bwd": [{"kernel": x["name"][:80], "us": x["gpu__time_duration.sum"] / 1e3,
                                   "dram_bytes": nbytes(x)} for x in group]},
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
