"""Exclusive vs shared device time per kernel group in a CUPTI trace of graph replays:
exclusive = time a group runs alone on the GPU (on the critical path for sure), shared =
overlapped time split evenly among the groups running.   python tools/r02/trace_share.py trace.json n_iters"""
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2510_00207_b200.timeline import kernel_group  # noqa: E402

ev = json.load(open(sys.argv[1]))
ev = ev["traceEvents"] if isinstance(ev, dict) else ev
n_it = int(sys.argv[2]) if len(sys.argv) > 2 else 20
k = [e for e in ev if e.get("cat") == "kernel" and "dur" in e]
evs = []
for e in k:
    g = kernel_group(e["name"])
    evs += [(e["ts"], 1, g), (e["ts"] + e["dur"], -1, g)]
evs.sort()
active, excl, shared, conc = collections.Counter(), collections.Counter(), collections.Counter(), collections.Counter()
idle, prev = 0.0, evs[0][0]
for t, d, g in evs:
    dt = t - prev
    if dt > 0:
        gs = [x for x, c in active.items() if c > 0]
        conc[min(len(gs), 3)] += dt
        if not gs:
            idle += dt
        elif len(gs) == 1:
            excl[gs[0]] += dt
        else:
            for x in gs:
                shared[x] += dt / len(gs)
    active[g] += d
    prev = t
span = evs[-1][0] - evs[0][0]
print(f"span {span / n_it:.1f} us/iter, idle {idle / n_it:.1f}, 1 group {conc[1] / n_it:.1f}, 2 groups {conc[2] / n_it:.1f}, 3+ {conc[3] / n_it:.1f}")
for g in sorted(set(excl) | set(shared), key=lambda g: -(excl[g] + shared[g])):
    print(f"{g:20s} exclusive {excl[g] / n_it:8.1f} us   shared(split) {shared[g] / n_it:8.1f} us")
