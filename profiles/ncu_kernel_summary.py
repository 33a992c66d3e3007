"""Key metrics of `ncu --set full` reports (one line per profiled kernel): duration,
tensor-pipe utilisation, DRAM bytes and DRAM throughput against peak.
Usage: python profiles/ncu_kernel_summary.py label=report.ncu-rep ... > profiles/rNN_ncu_kernels.txt"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("us", "gpu__time_duration.sum", 1e-3),
    ("tensor_pipe_%", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1),
    ("dram_GB", None, 1),
    ("dram_%peak", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("sm_%", "sm__throughput.avg.pct_of_peak_sustained_elapsed", 1),
    ("grid", "launch__grid_size", 1),
]


def rows(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        yield d, u


def num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return float("nan")


def main(args):
    print(f"{'label':28s} {'kernel':58s} {'us':>9s} {'tensor%':>8s} {'dram GB':>8s} {'dram%':>6s} {'sm%':>6s} {'grid':>6s}")
    for a in args:
        label, path = a.split("=", 1)
        for d, u in rows(path):
            scale = {"Mbyte": 1e-3, "Gbyte": 1.0, "Kbyte": 1e-6, "byte": 1e-9}
            rd = num(d.get("dram__bytes_read.sum", "nan")) * scale.get(u.get("dram__bytes_read.sum"), 1e-9)
            wr = num(d.get("dram__bytes_write.sum", "nan")) * scale.get(u.get("dram__bytes_write.sum"), 1e-9)
            t = num(d["gpu__time_duration.sum"]) * (1e-3 if u.get("gpu__time_duration.sum") == "nsecond" else 1.0)
            name = d["Kernel Name"].replace("void ", "")[:58]
            print(f"{label:28s} {name:58s} {t:9.2f} {num(d.get('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active','nan')):8.1f} "
                  f"{rd + wr:8.4f} {num(d.get('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed','nan')):6.1f} "
                  f"{num(d.get('sm__throughput.avg.pct_of_peak_sustained_elapsed','nan')):6.1f} {d.get('launch__grid_size','')[:6]:>6s}")


if __name__ == "__main__":
    main(sys.argv[1:])
