"""The schedule-property checker (paper_2510_00207_b200/schedule.py) on synthetic task
logs (no GPU): a schedule built in the paper's orders with every dependency honoured
passes; each kind of violation — an Eq.(3)-(6) order swap, a 6a-6e dependency broken, two
tasks overlapping on one stream, AR chunks out of order, an A2A held back while an AR chunk
starts — is reported.  PAPER.md P:198-253."""
import copy

from paper_2510_00207_b200.schedule import check_schedule, violations

COMP, A2A, AR = 1, 2, 3  # stream ids


def synth_log(L=2, R=2, P=2, dur=1.0):
    """List-schedule one iteration: compute tasks on stream COMP in Eq.(3)/(5) order, A2A
    tasks on A2A in Eq.(4)/(6) order, each starting at max(stream free, dependency end);
    AR chunks of a block after its AT^bwd on AR."""
    free = {COMP: 0.0, A2A: 0.0, AR: 0.0}
    end = {}
    recs = []

    def run(kind, block, chunk, d, stream, after=()):
        t0 = max([free[stream]] + [end[a] for a in after])
        t1 = t0 + dur
        free[stream] = t1
        end[(kind, block, chunk, d)] = t1
        recs.append(dict(kind=kind, block=block, chunk=chunk, dir=d, stream=stream, t0=t0, t1=t1))

    for b in range(L):  # forward, task-by-task in dependency-feasible order
        for r in range(R):
            run("AT", b, r, 0, COMP, [("MERGE", b - 1, r, 0)] if b else [])
        for r in range(R):
            run("D", b, r, 0, A2A, [("AT", b, r, 0)])
        for r in range(R):
            run("E", b, r, 0, COMP, [("D", b, r, 0)])
        for r in range(R):
            run("C", b, r, 0, A2A, [("E", b, r, 0)])
        for r in range(R):
            run("MERGE", b, r, 0, COMP, [("C", b, r, 0)])
    for cb in range(L):  # backward call cb = layer L-1-cb
        for r in reversed(range(R)):
            run("CBPACK", cb, r, 1, COMP, [("ATB", cb - 1, r, 1)] if cb else [])
        for r in reversed(range(R)):
            run("CB", cb, r, 1, A2A, [("CBPACK", cb, r, 1)])
        for r in reversed(range(R)):
            run("EB", cb, r, 1, COMP, [("CB", cb, r, 1)])
        for r in reversed(range(R)):
            run("DB", cb, r, 1, A2A, [("EB", cb, r, 1)])
        for r in reversed(range(R)):
            run("ATB", cb, r, 1, COMP, [("DB", cb, r, 1)])
        for c in range(3):
            run("AR", cb, c, 1, AR, [("ATB", cb, r, 1) for r in range(R)])
    return recs


def find(recs, kind, block, chunk, d):
    return next(r for r in recs if (r["kind"], r["block"], r["chunk"], r["dir"]) == (kind, block, chunk, d))


def test_valid_schedule_passes():
    recs = synth_log()
    res = check_schedule(recs, 2, 2, 2)
    assert violations(res) == {}, violations(res)
    for prop in ("eq3", "eq4", "eq5", "eq6", "6a", "6b", "6c", "6d", "6e", "stream_fifo", "ar_order"):
        assert res["checked"].get(prop, 0) > 0, prop


def test_p1_schedule_without_exchanges_passes():
    recs = [r for r in synth_log(P=1) if r["kind"] not in ("D", "C", "CB", "DB")]
    assert violations(check_schedule(recs, 2, 2, 1)) == {}


def test_order_swap_is_reported():
    recs = synth_log()
    a, b = find(recs, "AT", 0, 0, 0), find(recs, "AT", 0, 1, 0)
    a["t0"], b["t0"] = b["t0"], a["t0"]
    a["t1"], b["t1"] = b["t1"], a["t1"]
    assert "eq3" in violations(check_schedule(recs, 2, 2, 2))
    recs = synth_log()
    a, b = find(recs, "DB", 1, 1, 1), find(recs, "DB", 1, 0, 1)
    a["t0"], b["t0"] = b["t0"], a["t0"]
    a["t1"], b["t1"] = b["t1"], a["t1"]
    assert "eq6" in violations(check_schedule(recs, 2, 2, 2))


def test_broken_dependencies_are_reported():
    for kind, block, chunk, d, prop in (("EB", 0, 1, 1, "6b"), ("DB", 1, 0, 1, "6c"), ("ATB", 1, 1, 1, "6d"),
                                        ("CBPACK", 1, 0, 1, "6a"), ("E", 1, 0, 0, "fwd_E_after_D")):
        recs = synth_log()
        x = find(recs, kind, block, chunk, d)
        x["t0"] -= 1.5  # starts before its dependency ended
        v = violations(check_schedule(recs, 2, 2, 2))
        assert prop in v, (prop, v)
    recs = synth_log()
    ar = min((r for r in recs if r["kind"] == "AR" and r["block"] == 0), key=lambda r: r["t0"])
    ar["t0"] = find(recs, "ATB", 0, 0, 1)["t1"] - 0.5
    assert "6e" in violations(check_schedule(recs, 2, 2, 2))


def test_overlap_on_a_stream_and_ar_order_are_reported():
    recs = synth_log()
    x = find(recs, "MERGE", 0, 1, 0)
    x["t0"] -= 0.5  # overlaps the previous task on the compute stream
    assert "stream_fifo" in violations(check_schedule(recs, 2, 2, 2))
    recs = synth_log()
    a = [r for r in recs if r["kind"] == "AR" and r["block"] == 0]
    a[1]["chunk"], a[2]["chunk"] = 2, 1
    assert "ar_order" in violations(check_schedule(recs, 2, 2, 2))


def test_a2a_held_back_while_an_ar_chunk_starts_is_a_priority_violation():
    recs = synth_log()
    base = check_schedule(copy.deepcopy(recs), 2, 2, 2)
    assert base["priority_stats"]["held_back"] == 0 and base["priority_stats"]["a2a_tasks"] > 0
    # D^bwd of call 0 chunk 0 ready at end(EB) but started 1 ms later, and an AR chunk of
    # the same window started in between
    x = find(recs, "DB", 1, 0, 1)
    ready = find(recs, "EB", 1, 0, 1)["t1"]
    x["t0"] = ready + 1.0
    x["t1"] = x["t0"] + 1.0
    recs.append(dict(kind="AR", block=0, chunk=9, dir=1, stream=AR, t0=ready + 0.3, t1=ready + 0.6))
    res = check_schedule(recs, 2, 2, 2)
    assert res["priority_stats"]["held_back"] >= 1 and "priority" in violations(res)
