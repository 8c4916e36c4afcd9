"""Kernel timeline analysis from a CUPTI trace (torch.profiler chrome trace).

Measurement plumbing for bench.py (not part of the hot path):
  - per-kernel device time in the steady state (CUDA-graph replays),
  - idle time (no kernel on any stream of the GPU),
  - exposed communication: |∪ comm-kernel intervals \\ ∪ compute-kernel
    intervals|, reported as a fraction of total comm time and of the iteration time.
NCCL kernels are the comm kernels (A2A send/recv groups and AR chunks); everything else
on the device is compute.
"""
from __future__ import annotations

import collections
import json
import re


def _union(intervals):
    out = []
    for a, b in sorted(intervals):
        if out and a <= out[-1][1]:
            out[-1][1] = max(out[-1][1], b)
        else:
            out.append([a, b])
    return out


def _length(iv):
    return sum(b - a for a, b in iv)


def _subtract(a_iv, b_iv):
    """|A \\ B| for two sorted disjoint interval lists."""
    total, j = 0.0, 0
    for a0, a1 in a_iv:
        cur = a0
        while j < len(b_iv) and b_iv[j][1] <= cur:
            j += 1
        k = j
        while k < len(b_iv) and b_iv[k][0] < a1:
            b0, b1 = b_iv[k]
            if b0 > cur:
                total += b0 - cur
            cur = max(cur, b1)
            if cur >= a1:
                break
            k += 1
        if cur < a1:
            total += a1 - cur
    return total


def is_comm(name: str) -> bool:
    return (name.startswith("nccl") or "ncclDevKernel" in name or "ncclKernel" in name
            or "a2a_p2p" in name)


def short_name(name: str) -> str:
    n = re.sub(r"^void ", "", name)
    m = re.match(r"([\w:]+(?:<[^()]*?>)?)", n)
    return (m.group(1) if m else n)[:80]


# CUDA kernel name -> the kernel group the library's per-call-site profile uses
# (flowmoe_profile_* names: gemm_* -> "gemm", attn_fwd, attn_bwd, gate_topk, ...)
_GROUPS = (("gemm_tc_kernel", "gemm"), ("gemm_simt", "gemm"), ("attn_fwd", "attn_fwd"),
           ("attn_bwd", "attn_bwd"), ("gate_topk", "gate_topk"), ("gate_route", "gate_topk"),
           ("route_scan", "route_scan"), ("unpermute_combine", "unpermute_combine"),
           ("permute_pack", "permute_pack"), ("combine_bwd_pack", "combine_bwd_pack"),
           ("gather_gate_bwd", "gather_gate_bwd"), ("gate_wgrad", "gate_wgrad"), ("colsum", "colsum"),
           ("a2a_p2p", "a2a"), ("local_allreduce", "allreduce"))


def kernel_group(name: str) -> str:
    if is_comm(name) and "a2a_p2p" not in name:
        return "nccl"
    for needle, g in _GROUPS:
        if needle in name:
            return g
    return "other"


def analyze(trace_path: str, n_iters: int, trim: int = 0, a2a_bytes: float = 0.0, link_gbs: float = 770.0) -> dict:
    """Interval statistics of the traced kernels.  With trim > 0 the first and last
    `trim` iterations' worth of time are cut off (kernel intervals clipped to the
    middle window), so rank skew at the edges of the trace (NCCL kernels spinning
    on a late peer) does not count as exposed communication.

    A peer-memory exchange kernel copies first and then waits for the peers' arrivals; the
    wait is time spent on a slower peer (its compute or its copy), not on this rank's
    transfer.  With a2a_bytes (bytes one exchange moves over NVLink) the "transfer-only"
    exposure also counts each exchange kernel only over its first a2a_bytes / link_gbs."""
    ev = json.load(open(trace_path))
    ev = ev["traceEvents"] if isinstance(ev, dict) else ev
    kern = [e for e in ev if e.get("cat") == "kernel" and "dur" in e]
    if not kern:
        return {"error": "no kernel events in trace"}
    if trim > 0 and n_iters > 2 * trim:
        a = min(e["ts"] for e in kern)
        b = max(e["ts"] + e["dur"] for e in kern)
        it = (b - a) / n_iters
        lo, hi = a + trim * it, b - trim * it
        clipped = []
        for e in kern:
            s0, s1 = max(e["ts"], lo), min(e["ts"] + e["dur"], hi)
            if s1 > s0:
                clipped.append(dict(e, ts=s0, dur=s1 - s0))
        kern = clipped
        n_iters -= 2 * trim
    comm = [(e["ts"], e["ts"] + e["dur"]) for e in kern if is_comm(e["name"])]
    comp = [(e["ts"], e["ts"] + e["dur"]) for e in kern if not is_comm(e["name"])]
    uc, up = _union(comm), _union(comp)
    t0 = min(e["ts"] for e in kern)
    t1 = max(e["ts"] + e["dur"] for e in kern)
    busy = _union(comm + comp)
    per = collections.defaultdict(lambda: [0, 0.0])
    for e in kern:
        k = short_name(e["name"])
        per[k][0] += 1
        per[k][1] += e["dur"]
    by_group = collections.defaultdict(list)
    for e in kern:
        by_group[kernel_group(e["name"])].append((e["ts"], e["ts"] + e["dur"]))
    groups = {g: {"launches_per_iter": len(iv) / n_iters,
                  "sum_us_per_iter": sum(b - a for a, b in iv) / n_iters,
                  "busy_us_per_iter": _length(_union(iv)) / n_iters}
              for g, iv in by_group.items()}
    comm_us = _length(uc)
    exposed_us = _subtract(uc, up)
    xfer = []
    for e in kern:
        if not is_comm(e["name"]):
            continue
        d = e["dur"]
        if "a2a_p2p" in e["name"] and a2a_bytes > 0:
            d = min(d, a2a_bytes / (link_gbs * 1e3))  # bytes / (GB/s) in us
        xfer.append((e["ts"], e["ts"] + d))
    ux = _union(xfer)
    xfer_us, exposed_xfer_us = _length(ux), _subtract(ux, up)
    span_us = t1 - t0
    return {
        "iterations": n_iters,
        "span_us_per_iter": span_us / n_iters,
        "compute_busy_us_per_iter": _length(up) / n_iters,
        "comm_busy_us_per_iter": comm_us / n_iters,
        "exposed_comm_us_per_iter": exposed_us / n_iters,
        "exposed_comm_frac_of_comm": (exposed_us / comm_us) if comm_us > 0 else None,
        "exposed_comm_frac_of_iter": exposed_us / span_us if span_us > 0 else None,
        "idle_us_per_iter": (span_us - _length(busy)) / n_iters,
        "transfer_comm_us_per_iter": xfer_us / n_iters,
        "exposed_transfer_us_per_iter": exposed_xfer_us / n_iters,
        "exposed_transfer_frac_of_transfer": (exposed_xfer_us / xfer_us) if xfer_us > 0 else None,
        "kernels_per_iter": len(kern) / n_iters,
        "groups": groups,
        "top_kernels": sorted(([k, c // n_iters, d / n_iters] for k, (c, d) in per.items()),
                              key=lambda x: -x[2])[:25],
    }


def trace_replays(run, n_iters: int, path: str, trim: int = 0, sync=None, a2a_bytes: float = 0.0):
    """Run `run()` n_iters times under torch.profiler (CUDA activities) and write a chrome trace.
    `sync()` (e.g. a process-group barrier) runs once the profiler is live, so ranks whose
    CUPTI start-up took different times still enter the traced replays together."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        if sync is not None:
            sync()
            torch.cuda.synchronize()
        for _ in range(n_iters):
            run()
        torch.cuda.synchronize()
    prof.export_chrome_trace(path)
    return analyze(path, n_iters, trim, a2a_bytes=a2a_bytes)
