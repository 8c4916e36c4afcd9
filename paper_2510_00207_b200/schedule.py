"""Schedule properties of FlowMoE checked on a measured task log (flowmoe_tasklog_*).

Measurement plumbing (host-only, no method arithmetic): SURVEY §8(c.3) asks for the
schedule to be checked on measured timelines, since the paper prints no values to match:

  - Eq.(3)/(5): compute tasks in the order AT_1..AT_R, E_1..E_R per
    block forward, E_R..E_1, AT_R..AT_1 per block backward, blocks 1..L forward and L..1
    backward.  With one compute stream this is the total order of the compute tasks; with
    several compute lanes (a B200 addition) it holds on every lane.
  - Eq.(4)/(6): the A2A tasks D_1..D_R, C_1..C_R forward, C_R..C_1, D_R..D_1
    backward, per A2A stream.
  - 6a-6e: tau(C_r^(l-1)) >= end(AT_r^(l)), tau(E_r) >= end(C_r), tau(D_r) >=
    end(E_r), tau(AT_r) >= end(D_r), tau(AR^(l)) >= end(AT_r^(l)) for all r (backward),
    and the forward chain AT_r -> D_r -> E_r -> C_r -> merge.
  - one stream runs one task at a time (no overlap within a stream, P:227's resource model
    per stream).
  - AR chunks of a block in flat-buffer order, blocks L..1 (reading Q11).
  - the priority rule ("at every comm dispatch with a nonempty A2A
    queue the dispatched task is an A2A task").  On B200 the AR chunks run on their own
    low-priority stream and communicator next to the A2As rather than in one FIFO comm
    resource, so the measurable form is: no A2A task is held back past its
    ready time while an AR chunk starts in the gap.  ready(A2A) = the later of its
    dependency's end and the end of the previous task on its stream.

Task records are dicts with kind (flowmoe.TASK_KINDS), block (call index per direction),
chunk (r, or -1 for an unsplit AT / the wgrad tasks / AR chunk index for AR), dir (0 fwd,
1 bwd), stream, t0, t1 (ms).
"""
from __future__ import annotations

import collections

A2A = ("D", "C", "CB", "DB")


def _by(recs, **kw):
    return [r for r in recs if all(r[k] == v for k, v in kw.items())]


def check_schedule(recs: list, L: int, R: int, P: int, eps_ms: float = 0.002, prio_eps_ms: float = 0.005) -> dict:
    """All properties above on one rank's task log of an L-block iteration (fwd + bwd).
    Returns {property: [violations]} plus 'checked' counts and 'priority' statistics."""
    out = collections.defaultdict(list)
    checked = collections.Counter()
    fwd = [r for r in recs if r["dir"] == 0]
    bwd = [r for r in recs if r["dir"] == 1]

    def layer_b(r):  # backward call index -> stack layer (blocks run L-1 .. 0)
        return L - 1 - r["block"]

    # ---- no overlap within a stream
    by_stream = collections.defaultdict(list)
    for r in recs:
        by_stream[r["stream"]].append(r)
    for s, rs in by_stream.items():
        rs = sorted(rs, key=lambda r: (r["t0"], r["t1"]))
        for a, b in zip(rs, rs[1:]):
            checked["stream_fifo"] += 1
            if b["t0"] < a["t1"] - eps_ms:
                out["stream_fifo"].append((a["kind"], a["block"], a["chunk"], b["kind"], b["block"], b["chunk"]))

    # ---- Eq.(3)-(6) orders, per stream
    def rank(r):
        c = r["chunk"]
        if r["dir"] == 0:
            base = r["block"] * 2 * R
            return {"AT": base + max(c, 0), "E": base + R + c, "D": base + c, "C": base + R + c}.get(r["kind"])
        base = (L - 1 - layer_b(r)) * 2 * R
        rc = R - 1 - c if c >= 0 else R - 1
        return {"EB": base + rc, "ATB": base + R + rc, "CB": base + rc, "DB": base + R + rc}.get(r["kind"])

    for name, kinds, d in (("eq3", ("AT", "E"), 0), ("eq4", ("D", "C"), 0),
                           ("eq5", ("EB", "ATB"), 1), ("eq6", ("CB", "DB"), 1)):
        for s, rs in by_stream.items():
            seq = sorted((r for r in rs if r["kind"] in kinds and r["dir"] == d), key=lambda r: r["t0"])
            for a, b in zip(seq, seq[1:]):
                checked[name] += 1
                if rank(b) < rank(a):
                    out[name].append((a["kind"], a["block"], a["chunk"], b["kind"], b["block"], b["chunk"]))

    # ---- forward chain AT_r -> D_r -> E_r -> C_r -> merge (P = 1: AT_r -> E_r -> merge)
    def one(rs, kind, block, chunk, d):
        m = [r for r in rs if r["kind"] == kind and r["block"] == block and r["dir"] == d and
             (r["chunk"] == chunk or (kind in ("AT", "ATB") and r["chunk"] == -1))]
        return m[0] if m else None

    def dep(name, later, earlier):
        if later is None or earlier is None:
            return
        checked[name] += 1
        if later["t0"] < earlier["t1"] - eps_ms:
            out[name].append((later["kind"], later["block"], later["chunk"], earlier["kind"], earlier["block"],
                              earlier["chunk"], round(earlier["t1"] - later["t0"], 5)))

    for b in range(L):
        for r in range(R):
            at = one(fwd, "AT", b, r, 0)
            d = one(fwd, "D", b, r, 0) if P > 1 else None
            e = one(fwd, "E", b, r, 0)
            c = one(fwd, "C", b, r, 0) if P > 1 else None
            m = one(fwd, "MERGE", b, r, 0)
            if P > 1:
                dep("fwd_D_after_AT", d, at)
                dep("fwd_E_after_D", e, d)
                dep("fwd_C_after_E", c, e)
                dep("fwd_merge_after_C", m, c)
            else:
                dep("fwd_E_after_AT", e, at)
                dep("fwd_merge_after_E", m, e)
            if b + 1 < L:
                dep("fwd_next_AT_after_merge", one(fwd, "AT", b + 1, r, 0), m)

    # ---- backward 6a-6e (call index cb = L-1-l)
    for cb in range(L):
        for r in range(R):
            cpack = one(bwd, "CBPACK", cb, r, 1)
            c = one(bwd, "CB", cb, r, 1) if P > 1 else cpack
            e = one(bwd, "EB", cb, r, 1)
            d = one(bwd, "DB", cb, r, 1) if P > 1 else None
            at = one(bwd, "ATB", cb, r, 1)
            if cb + 1 < L:  # 6a: C_r of the next block backward (l-1) after AT_r of this one (l)
                dep("6a", one(bwd, "CBPACK", cb + 1, r, 1), at)
            dep("6b", e, c)
            if P > 1:
                dep("6c", d, e)
                dep("6d", at, d)
            else:
                dep("6d", at, e)
        ars = sorted(_by(bwd, kind="AR", block=cb), key=lambda r: r["t0"])
        ats = _by(bwd, kind="ATB", block=cb)
        if ars and ats:
            last_at = max(ats, key=lambda r: r["t1"])
            dep("6e", ars[0], last_at)
            # AR chunks of the block in flat-buffer order (reading Q11); two parameter groups
            # ([dWo|dWg] first, then dWqkv) each restart the chunk index at 0
            for a, b2 in zip(ars, ars[1:]):
                checked["ar_order"] += 1
                if b2["chunk"] < a["chunk"] and b2["chunk"] != 0:
                    out["ar_order"].append((cb, a["chunk"], b2["chunk"]))
    # blocks L..1: every AR chunk of call cb starts before any of call cb+1 (same AR stream)
    ar_all = [r for r in bwd if r["kind"] == "AR"]
    for cb in range(L - 1):
        a = [r["t0"] for r in ar_all if r["block"] == cb]
        b = [r["t0"] for r in ar_all if r["block"] == cb + 1]
        if a and b:
            checked["ar_block_order"] += 1
            if min(b) < max(a) - eps_ms:
                out["ar_block_order"].append((cb, cb + 1))

    # ---- priority: an AR chunk never starts while a ready A2A task is held back
    prio = {"a2a_tasks": 0, "held_back": 0, "max_hold_ms": 0.0}
    if P > 1:
        ar_starts = sorted(r["t0"] for r in recs if r["kind"] == "AR")
        deps = {"D": ("AT", 0), "C": ("E", 0), "CB": ("CBPACK", 1), "DB": ("EB", 1)}
        for x in recs:
            if x["kind"] not in A2A:
                continue
            pk, d = deps[x["kind"]]
            pre = one(fwd if d == 0 else bwd, pk, x["block"], x["chunk"], d)
            if pre is None:
                continue
            prev = [r["t1"] for r in by_stream[x["stream"]] if r["t1"] <= x["t0"] + eps_ms and r is not x]
            ready = max([pre["t1"]] + ([max(prev)] if prev else []))
            hold = x["t0"] - ready
            prio["a2a_tasks"] += 1
            prio["max_hold_ms"] = max(prio["max_hold_ms"], hold)
            if hold > prio_eps_ms and any(ready < t < x["t0"] for t in ar_starts):
                prio["held_back"] += 1
                out["priority"].append((x["kind"], x["block"], x["chunk"], round(hold, 5)))
        checked["priority"] = prio["a2a_tasks"]
    res = {k: v for k, v in out.items()}
    res["checked"] = dict(checked)
    res["priority_stats"] = prio
    return res


def violations(res: dict, ignore=()) -> dict:
    """The non-empty violation lists of check_schedule's result."""
    return {k: v for k, v in res.items() if k not in ("checked", "priority_stats") and v and k not in ignore}
