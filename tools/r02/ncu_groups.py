"""Summarise an ncu --csv metrics list of a bench run by kernel group (timeline.kernel_group):
launches, device time (cold-cache, serialised: compare SHARES), DRAM bytes per launch, and for
the GEMM the tcgen05 tensor-pipe utilisation from the UTCHMMA instruction count:
  util = Σ UTCHMMA · busy cycles per instruction · SMs per instruction / (cycles · 148)
(M=128 x N=BN 1-CTA: BN/2 cycles on 1 SM; M=256 x N=256 pair: 128 cycles on 2 SMs).
Updates profiles/ncu_traffic.json[config][group].
  python tools/r02/ncu_groups.py launches.csv config > summary.md"""
import collections
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from paper_2510_00207_b200.timeline import kernel_group  # noqa: E402


def main(path, config):
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, mi, vi, ii = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    per = collections.OrderedDict()
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        d = per.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", "") or 0)
    agg = collections.defaultdict(lambda: collections.Counter())
    for d in per.values():
        g = kernel_group(d["name"])
        if g == "other":
            continue
        a = agg[g]
        a["launches"] += 1
        a["us"] += d.get("gpu__time_duration.sum", 0) / 1e3
        a["dram"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
        if g == "gemm":
            m = re.search(r"gemm_tc_kernel<(\d+), \d+, \d+, (\d+)>", d["name"]) or re.search(r"gemm_tc_kernel<(\d+)", d["name"])
            bn = int(m.group(1)) if m else 256
            cg = int(m.group(2)) if m and m.lastindex >= 2 else 1
            n = d.get("sm__inst_executed_pipe_tensor_subpipe_hmma.sum", 0)
            busy = n * (bn / 2 if cg == 1 else bn * 256 / 512) * (1 if cg == 1 else 2)  # SM-cycles
            cyc = d.get("gpu__time_duration.sum", 0) * 1e-9 * d.get("sm__cycles_elapsed.avg.per_second", 0)
            a["tc_busy"] += busy
            a["tc_avail"] += cyc * 148
    tot = sum(a["us"] for a in agg.values())
    print(f"# ncu launch list by kernel group — {config} ({path})\n")
    print("| group | launches | µs total | share | µs / launch | DRAM MB / launch | tensor-pipe util |")
    print("|---|---|---|---|---|---|---|")
    tr_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    tr = json.load(open(tr_path)) if os.path.exists(tr_path) else {}
    cur = tr.setdefault(config, {})
    for g, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        util = a["tc_busy"] / a["tc_avail"] if a.get("tc_avail") else None
        print(f"| {g} | {a['launches']} | {a['us']:.1f} | {a['us'] / tot:.3f} | {a['us'] / a['launches']:.1f} | "
              f"{a['dram'] / a['launches'] / 1e6:.2f} | {'' if util is None else f'{util:.3f}'} |")
        cur[g] = {"launches": a["launches"], "us_per_launch": a["us"] / a["launches"],
                  "dram_bytes_per_launch": a["dram"] / a["launches"], "share_of_listed": a["us"] / tot,
                  "tensor_pipe_util": util, "source": os.path.basename(path)}
    json.dump(tr, open(tr_path, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
