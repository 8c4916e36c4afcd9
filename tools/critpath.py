"""Critical-path view of one CUDA-graph replay from a CUPTI chrome trace (bench.py
--trace-dir): for the kernels of one iteration, walk back from the last-ending kernel,
each step taking the latest-ending kernel that ended before this one started (PDL lets
a kernel start before its predecessor ends, so also consider kernels ending before
this one's end that started earlier).  Prints per-kernel-name time on that chain."""
import collections
import gzip
import json
import re
import sys


def short(n):
    n = re.sub(r"^void ", "", n)
    m = re.match(r"([\w:]+(?:<[^()]*?>)?)", n)
    return (m.group(1) if m else n)[:48]


def main(path, n_iters=6, it=2):
    ev = json.load(gzip.open(path) if path.endswith(".gz") else open(path))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    k = sorted((e for e in ev if e.get("cat") == "kernel"), key=lambda e: e["ts"])
    t0, t1 = k[0]["ts"], max(e["ts"] + e["dur"] for e in k)
    span = (t1 - t0) / n_iters
    lo, hi = t0 + it * span, t0 + (it + 1) * span
    win = [e for e in k if lo <= e["ts"] < hi]
    ends = sorted(win, key=lambda e: e["ts"] + e["dur"])
    cur = ends[-1]
    chain = [cur]
    while True:
        # predecessor: latest-ending kernel that ended before cur ended and started before cur
        cands = [e for e in ends if e["ts"] + e["dur"] <= cur["ts"] + cur["dur"] - 1e-6 and e["ts"] < cur["ts"]
                 and e is not cur]
        if not cands:
            break
        prv = max(cands, key=lambda e: e["ts"] + e["dur"])
        if prv["ts"] + prv["dur"] < lo:
            break
        chain.append(prv)
        cur = prv
    chain.reverse()
    per = collections.defaultdict(lambda: [0, 0.0])
    for a, b in zip(chain, chain[1:] + [None]):
        end_a = a["ts"] + a["dur"]
        inc = (b["ts"] + b["dur"] - end_a) if b else 0.0  # time the chain advanced while b ran
        if b:
            p = per[short(b["name"])]
            p[0] += 1
            p[1] += inc
    tot = sum(v[1] for v in per.values())
    print(f"iteration span {span:.1f} us; chain {len(chain)} kernels, {tot:.1f} us")
    for n, (c, t) in sorted(per.items(), key=lambda x: -x[1][1]):
        print(f"  {n:48s} {c:4d}  {t:8.1f} us  {t / c:6.2f} us/each")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 6)
