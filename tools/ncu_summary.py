"""Summarise ncu captures into profiles/: per-kernel-function launch count, mean device
time and DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) per launch.
Usage: python tools/ncu_summary.py <report.ncu-rep | metrics.csv> <config> [--traffic-json profiles/ncu_traffic.json]
"""
import collections
import csv
import io
import json
import re
import subprocess
import sys


def rows_from(path):
    if path.endswith(".ncu-rep"):
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--metrics",
                              "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"],
                             capture_output=True, text=True).stdout
        rd = list(csv.reader(io.StringIO(out)))
        hdr, units, data = rd[0], rd[1], rd[2:]
        idx = {h: i for i, h in enumerate(hdr)}
        scale = {}
        for m in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
            u = units[idx[m]]
            scale[m] = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3,
                        "s": 1e6, "second": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                        "Tbyte": 1e12}.get(u, 1.0)
        for r in data:
            yield (r[idx["Kernel Name"]], float(r[idx["gpu__time_duration.sum"]]) * scale["gpu__time_duration.sum"],
                   float(r[idx["dram__bytes_read.sum"]]) * scale["dram__bytes_read.sum"]
                   + float(r[idx["dram__bytes_write.sum"]]) * scale["dram__bytes_write.sum"])
    else:  # --csv --log-file of a --metrics run: one row per (launch, metric)
        lines = [l for l in open(path) if not l.startswith("==")]
        per = collections.OrderedDict()
        for r in csv.DictReader(io.StringIO("".join(lines))):
            key = r["ID"]
            d = per.setdefault(key, {"name": r["Kernel Name"], "t": 0.0, "b": 0.0})
            v = float(r["Metric Value"].replace(",", ""))
            u = r["Metric Unit"]
            if r["Metric Name"] == "gpu__time_duration.sum":
                d["t"] = v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1e-3)
            elif r["Metric Name"].startswith("dram__bytes"):
                d["b"] += v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
        for d in per.values():
            yield d["name"], d["t"], d["b"]


def fn_name(n):
    n = re.sub(r"^void ", "", n)
    n = re.sub(r"^fm::", "", n)
    m = re.match(r"(\w+)", n)
    return m.group(1) if m else n


if __name__ == "__main__":
    path, config = sys.argv[1], sys.argv[2]
    agg = collections.OrderedDict()
    for name, t_us, b in rows_from(path):
        a = agg.setdefault(fn_name(name), [0, 0.0, 0.0])
        a[0] += 1
        a[1] += t_us
        a[2] += b
    print(f"{'kernel':32s} {'launches':>8s} {'mean_us':>9s} {'dram_MB/launch':>15s} {'GB/s':>8s}")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:32s} {n:8d} {t / n:9.2f} {b / n / 1e6:15.3f} {b / (t * 1e-6) / 1e9 if t else 0:8.1f}")
    if "--traffic-json" in sys.argv:
        out = sys.argv[sys.argv.index("--traffic-json") + 1]
        try:
            tr = json.load(open(out))
        except Exception:
            tr = {}
        ent = tr.setdefault(config, {})
        for k, (n, t, b) in agg.items():
            key = "gemm_tc (all calls)" if k == "gemm_tc_kernel" else k
            ent[key] = {"dram_bytes_per_launch": b / n, "mean_us": t / n, "launches": n, "source": path.split("/")[-1]}
        json.dump(tr, open(out, "w"), indent=1)
