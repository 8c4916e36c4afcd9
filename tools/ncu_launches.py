"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel
count, total and per-launch device time, and share of the listed time."""
import collections
import csv
import io
import re
import sys


def load(path):
    lines = [l for l in open(path) if not l.startswith("==")]
    rows = [r for r in csv.DictReader(io.StringIO("".join(lines))) if r.get("Metric Name") == "gpu__time_duration.sum"]
    return rows


def short(n):
    n = re.sub(r"^void ", "", n)
    m = re.match(r"([\w:]+(?:<[^()]*?>)?)", n)
    s = m.group(1) if m else n
    return s[:70]


def summarise(path, skip_prefix=("at::", "(anonymous", "void at::")):
    rows = load(path)
    agg = collections.OrderedDict()
    for r in rows:
        n = short(r["Kernel Name"])
        t = float(r["Metric Value"]) / 1000.0
        a = agg.setdefault(n, [0, 0.0])
        a[0] += 1
        a[1] += t
    tot = sum(v[1] for k, v in agg.items() if not k.startswith(skip_prefix))
    out = []
    for n, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append((n, c, t, t / c, t / tot if not n.startswith(skip_prefix) else 0.0))
    return out, tot


if __name__ == "__main__":
    out, tot = summarise(sys.argv[1])
    print(f"{'kernel':70s} {'n':>5s} {'total_us':>10s} {'per_us':>8s} {'share':>6s}")
    for n, c, t, per, sh in out[:40]:
        print(f"{n:70s} {c:5d} {t:10.1f} {per:8.2f} {sh:6.3f}")
    print("flowmoe kernels total us:", round(tot, 1))
