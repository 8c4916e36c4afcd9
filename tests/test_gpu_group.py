"""The exchange rows on ONE GPU: P ranks in the in-process simulated world
(flowmoe_create_local_group, include/flowmoe_test.h).  The ranks' buffers live on the same
device, the real peer-memory A2A kernels move the dispatch / combine blocks between them
(S6 D_r, S8 C_r, B1 C_r^bwd, B3 D_r^bwd: owner side [E][R][C][M] <-> expert side
[E/P][R][P][C][M], arrival counters advancing over repeated iterations), and the all-reduce
of the MHA + gate grads runs the S_p chunk loop (B6, Alg. 2 PARTITION P:319-324).  Each
rank is driven by its own host thread; the ranks never spin on each other on the device
(their exchanges meet at host barriers and order the streams with events).  Checked
against the oracle's P simulated workers exactly like the multi-GPU test (PAPER.md P:17,
P:207)."""
import numpy as np
import pytest

import oracle as o
from synth import PRESETS, BlockConfig, gen_replicated, gen_worker
from tests.gpu_util import chain_per_block_errors, expert_grads, oracle_block, rel, run_group_gpu

pytestmark = pytest.mark.gpu
TOL = {"f32": 1e-4, "bf16": 2e-2}

CASES = {
    "c1_f32": PRESETS["c1"],
    "bf16_p": BlockConfig(T=512, seq_len=128, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=2,
                          capacity_factor=1.0, causal=1, residual=1, dtype="bf16"),
    "bf16_tok": BlockConfig(T=512, seq_len=512, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=4,
                            capacity_factor=1.0, causal=1, residual=1, dtype="bf16"),
    "bf16_k3_drop": BlockConfig(T=384, seq_len=96, M=192, n_heads=3, E=8, top_k=3, d_ffn=328, R=2,
                                capacity_factor=0.75, causal=0, residual=0, dtype="bf16"),
}


def _check(name, P, lanes, schedule="flowmoe", chunk_bytes=4096 + 16):
    cfg = CASES[name].replace(P=P)
    rep = gen_replicated(cfg)
    wks = [gen_worker(cfg, p) for p in range(P)]
    repeat = 2
    gs = run_group_gpu(cfg, rep, wks, chunk_bytes=chunk_bytes, compute_streams=lanes, schedule=schedule,
                       repeat=repeat)
    ys, dxs, gflat, eg, st = oracle_block(cfg, rep, wks)
    El = cfg.E // P
    tol = TOL[cfg.dtype]
    for q, g in enumerate(gs):
        res = {"y": rel(g["y"], ys[q]), "dx": rel(g["dx"], dxs[q]), "grad_flat": rel(g["grad_flat"], gflat)}
        ref_e = expert_grads(eg, q * El, (q + 1) * El)
        for n in ("dw1", "db1", "dw2", "db2"):
            res[n] = rel(g[n], ref_e[n])
        bad = {k: v for k, v in res.items() if not v <= tol}
        assert not bad, (q, bad, res)
        ro = st.route[q]
        assert np.array_equal(g["idx"], ro.idx), q
        assert np.array_equal(g["pos"], np.where(ro.kept, ro.pos, -1)), q
        assert np.array_equal(g["counts"], ro.counts), q
    # the all-reduced replicated grads are the same sum on every rank, bit for bit
    for g in gs[1:]:
        assert np.array_equal(g["grad_flat"], gs[0]["grad_flat"])
    # every source delivered each of the 4 exchanges of every chunk once per iteration
    for g in gs:
        assert np.all(g["arrivals"] == repeat), g["arrivals"]
    return gs


@pytest.mark.parametrize("P", [2, 4])
@pytest.mark.parametrize("name", ["c1_f32", "bf16_p", "bf16_k3_drop"])
def test_local_group_block_parity(name, P):
    """Block fwd+bwd on P simulated ranks vs the oracle's P workers (forced routing),
    two iterations (the A2A arrival counters and `seen` epochs advance), a tiny S_p so the
    AR is cut into many chunks plus a remainder."""
    _check(name, P, lanes=CASES[name].R)


@pytest.mark.parametrize("name", ["bf16_p", "bf16_k3_drop"])
def test_local_group_block_parity_eight_ranks(name):
    """P = 8 (one expert per rank, the largest world the peer-memory A2A supports and the
    driver's 8-GPU scaling point): the same checks on eight simulated ranks."""
    _check(name, 8, lanes=CASES[name].R)


def test_local_group_one_lane_and_flowmoe_ar():
    """The paper's single compute stream, and the FLOWMOE_AR policy (AT unsplit)."""
    _check("bf16_p", 2, lanes=1)
    _check("bf16_p", 2, lanes=2, schedule="flowmoe_ar")


def test_local_group_token_chunks():
    """Token chunks (reading Q1') with the exchanges: R = 4 causal slices of one sequence."""
    _check("bf16_tok", 2, lanes=4)


def test_local_group_stack_per_block_parity():
    """A 3-block stack through flowmoe_stack_fwd/bwd on 2 simulated ranks (lanes forked once,
    the exchanges of chunk r of block l+1 right behind block l): every block vs the oracle's
    2 workers on that block's GPU inputs; arrival counters = iterations x blocks."""
    cfg = CASES["bf16_p"].replace(P=2)
    L, P = 3, 2
    reps = [gen_replicated(cfg, block=l) for l in range(L)]
    wks = [gen_worker(cfg, p) for p in range(P)]
    gs = run_group_gpu(cfg, None, wks, compute_streams=cfg.R, stack_reps=reps, repeat=2)
    for g in gs:
        assert np.all(g["arrivals"] == 2 * L), g["arrivals"]
    for g in gs:
        g["grad_flat"], g["dw1"] = g["grad_flat_l"], g["dw1_l"]
    forced = [[w["forced_idx"]] * L for w in wks]
    for q in range(P):
        res = chain_per_block_errors(cfg, reps, forced, [w["dy"] for w in wks], gs, rank=q, P=P)
        bad = {k: v for k, v in res.items() if not v <= TOL["bf16"]}
        assert not bad, (q, bad, res)


@pytest.mark.parametrize("P", [2, 4, 8])
@pytest.mark.parametrize("s_p", [16, 4096 + 16, 1 << 20, 1 << 30])
def test_local_group_chunked_allreduce_matches_oracle(P, s_p):
    """flowmoe_allreduce_submit on P simulated ranks: the S_p partition (chunks of S_p plus
    a remainder) summed chunk by chunk in rank order == oracle.allreduce_chunked,
    bit for bit in fp32 (random data: the sums round), on every rank; and one all-reduce
    kernel per chunk of oracle.partition_ar."""
    import torch
    import paper_2510_00207_b200 as fm
    from tests.gpu_util import shape_of
    cfg = (CASES["c1_f32"] if P <= 4 else CASES["bf16_p"].replace(dtype="f32")).replace(P=P)  # E % P == 0
    ctxs = fm.FlowMoE.local_group(shape_of(cfg, P, 0, "overwrite", 1, "flowmoe", "p2p"), P, 0)
    n = 100_003  # odd: every S_p leaves a remainder chunk
    rng = np.random.default_rng(P * 31 + s_p % 97)
    host = [rng.standard_normal(n).astype(np.float32) for _ in range(P)]
    dev = [torch.from_numpy(h).cuda() for h in host]
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()
    n0 = fm.kernel_launches()
    tickets = [ctxs[q].allreduce_submit(dev[q], n, s_p) for q in range(P)]
    launched = fm.kernel_launches() - n0
    for q in range(P):
        ctxs[q].allreduce_wait(tickets[q], s)
    torch.cuda.synchronize()
    want = o.allreduce_chunked(host, s_p // 4, np.float32)
    for q in range(P):
        assert np.array_equal(dev[q].cpu().numpy(), want), q
    assert launched == len(o.partition_ar(4 * n, s_p))
    for c in ctxs:
        c.close()


def test_local_group_wait_before_peers_submit_is_an_error():
    """allreduce_wait on a ticket whose peers have not submitted yet: FLOWMOE_ERR_STATE
    (the simulated world cannot run a rank's all-reduce alone)."""
    import torch
    import paper_2510_00207_b200 as fm
    from tests.gpu_util import shape_of
    cfg = CASES["c1_f32"]
    ctxs = fm.FlowMoE.local_group(shape_of(cfg, 2, 0, "overwrite", 1, "flowmoe", "p2p"), 2, 0)
    a = torch.zeros(1000, device="cuda")
    b = torch.ones(1000, device="cuda")
    t0 = ctxs[0].allreduce_submit(a, 1000, 1024)
    with pytest.raises(fm.FlowMoEError, match="invalid state"):
        ctxs[0].allreduce_wait(t0, torch.cuda.current_stream())
    t1 = ctxs[1].allreduce_submit(b, 1000, 1024)
    ctxs[0].allreduce_wait(t0, torch.cuda.current_stream())
    ctxs[1].allreduce_wait(t1, torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert torch.all(a == 1) and torch.all(b == 1)
    for c in ctxs:
        c.close()
