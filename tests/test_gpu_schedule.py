"""Schedule properties on measured timelines: the task log of one eager
iteration of an L-block stack (flowmoe_tasklog_*, include/flowmoe_test.h) is checked for
the Eq.(3)/(5) compute orders, the Eq.(4)/(6) A2A orders, the 6a-6e dependencies (PAPER.md
P:198-242), one task at a time per stream, the AR chunk order (reading Q11) and the
A2A-before-AR priority rule — on one GPU at P = 1 and on two
simulated ranks (the exchange tasks present), in the paper's single-compute-stream
schedule and with several compute lanes."""
import threading

import pytest

import paper_2510_00207_b200 as fm
from paper_2510_00207_b200.schedule import check_schedule, violations
from synth import BlockConfig, gen_replicated, gen_worker
from tests.gpu_util import shape_of

pytestmark = pytest.mark.gpu

CFG = BlockConfig(T=1024, seq_len=256, M=512, n_heads=4, E=8, top_k=2, d_ffn=1024, R=4,
                  capacity_factor=1.0, causal=1, residual=1, dtype="bf16")


def stack_logs(cfg, P, lanes, L=3, schedule="flowmoe", chunk_bytes=256 << 10):
    """Task logs (one per rank) of one eager L-block iteration (stack API), after a warm-up
    iteration; P > 1 runs the simulated world, one host thread per rank."""
    import torch
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfgp = cfg.replace(P=P)
    shape = shape_of(cfgp, P, 0, "overwrite", lanes, schedule, "p2p" if P > 1 else "nccl")
    ctxs = fm.FlowMoE.local_group(shape, P, 0) if P > 1 else [fm.FlowMoE(shape, 0, None)]
    reps = [gen_replicated(cfgp, block=l) for l in range(L)]
    bts = [[fm.BlockTensors(r, cfg.dtype, q, P, dev) for r in reps] for q in range(P)]
    wks = [gen_worker(cfgp, q) for q in range(P)]
    xs = [[fm.to_device(wks[q]["x"], cfg.dtype, dev)] + [None] * L for q in range(P)]
    for q in range(P):
        for l in range(L):
            xs[q][l + 1] = torch.empty_like(xs[q][0])
    dxs = [[torch.empty_like(xs[q][0]) for _ in range(L)] for q in range(P)]
    dys = [fm.to_device(wks[q]["dy"], cfg.dtype, dev) for q in range(P)]
    saved = [[torch.empty(ctxs[q].saved_bytes, dtype=torch.uint8, device=dev) for _ in range(L)] for q in range(P)]
    for l in range(L):
        for q in range(P):
            ctxs[q].register_saved(saved[q][l])
    s = torch.cuda.current_stream()

    def iteration(q, tickets, errs):
        try:
            ctxs[q].stack_fwd([b.params for b in bts[q]], xs[q][0], xs[q][1:], saved[q], s)
            tickets[q] = ctxs[q].stack_bwd([b.params for b in bts[q]], xs[q][0], xs[q][1:], saved[q], dys[q],
                                           dxs[q], [b.grads for b in bts[q]], chunk_bytes, s)
        except BaseException as e:  # re-raised by the caller
            errs[q] = e

    def run_all():
        tickets, errs = [None] * P, [None] * P
        th = [threading.Thread(target=iteration, args=(q, tickets, errs)) for q in range(P)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        for e in errs:
            if e is not None:
                raise e
        for q in range(P):
            for t in tickets[q]:
                ctxs[q].allreduce_wait(t, s)

    run_all()  # warm-up (modules loaded, stashes registered)
    torch.cuda.synchronize()
    for c in ctxs:
        c.tasklog_begin()
    if P == 1:  # the whole iteration enqueued before the GPU starts it (no host gaps)
        from tests.gpu_util import HostGate
        gate = HostGate(s)
        run_all()
        gate.release()
    else:  # the simulated ranks' host threads meet at barriers: they cannot all enqueue first
        run_all()
    logs = [c.tasklog_end() for c in ctxs]
    for c in ctxs:
        c.close()
    return logs


@pytest.mark.parametrize("lanes", [1, 4])
def test_schedule_properties_one_rank(lanes):
    L = 3
    (log,) = stack_logs(CFG, 1, lanes, L)
    kinds = {r["kind"] for r in log}
    assert {"AT", "E", "MERGE", "CBPACK", "EB", "ATB", "WGE", "WGA"} <= kinds, kinds
    assert sum(r["kind"] == "AT" for r in log) == L * CFG.R
    res = check_schedule(log, L, CFG.R, 1)
    assert violations(res) == {}, violations(res)
    for prop in ("eq3", "eq5", "6a", "6b", "6d", "stream_fifo", "fwd_E_after_AT"):
        assert res["checked"].get(prop, 0) > 0, (prop, res["checked"])
    if lanes == 1:  # the paper's single compute stream: Eq.(3) is the total order
        comp = sorted((r for r in log if r["kind"] in ("AT", "E") and r["dir"] == 0), key=lambda r: r["t0"])
        want = [(k, b, c) for b in range(L) for k in ("AT", "E") for c in range(CFG.R)]
        assert [(r["kind"], r["block"], r["chunk"]) for r in comp] == want


@pytest.mark.parametrize("lanes", [1, 2])
def test_schedule_properties_two_simulated_ranks(lanes):
    """P = 2 in the simulated world: the A2A tasks (D, C, C^bwd, D^bwd exchanges) and the
    chunked AR (S_p = 256 KiB: several chunks per block) are in the log; Eq.(4)/(6),
    6a-6e including the exchanges, and the AR after every AT^bwd of its block.  The
    priority rule is only reported here (the ranks' host threads meet at barriers, so a
    host-side delay can look like a held-back A2A); the multi-GPU test asserts it."""
    L = 3
    logs = stack_logs(CFG, 2, lanes, L)
    for q, log in enumerate(logs):
        kinds = {r["kind"] for r in log}
        assert {"D", "C", "CB", "DB", "AR"} <= kinds, kinds
        res = check_schedule(log, L, CFG.R, 2)
        v = violations(res, ignore=("priority",))
        assert v == {}, (q, v)
        for prop in ("eq4", "eq6", "6c", "6e", "fwd_D_after_AT", "fwd_C_after_E", "ar_order"):
            assert res["checked"].get(prop, 0) > 0, (q, prop, res["checked"])
        print("rank", q, "priority", res["priority_stats"])
