"""One rank of the multi-GPU parity check (launched by tests/test_gpu_multi.py via
torchrun).  Every rank runs its block through the C ABI with world_size = P and
compares its own outputs with the oracle's P simulated workers."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import oracle as o  # noqa: E402
import paper_2510_00207_b200 as fm  # noqa: E402
from synth import PRESETS, BlockConfig, gen_replicated, gen_worker  # noqa: E402
from tests.gpu_util import (chain_per_block_errors, expert_grads, oracle_block, rel,  # noqa: E402
                            run_block_gpu, run_stack_gpu)

CASES = {
    "c1_f32": PRESETS["c1"],
    "bf16_p": BlockConfig(T=512, seq_len=128, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=2,
                          capacity_factor=1.0, causal=1, residual=1, dtype="bf16"),
    # token chunks (reading Q1'): 4 causal slices of one 512-token sequence
    "bf16_tok": BlockConfig(T=512, seq_len=512, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=4,
                            capacity_factor=1.0, causal=1, residual=1, dtype="bf16"),
}


def main():
    rank = int(os.environ["RANK"])
    P = int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    results = {}
    runs = [(n, c, "flowmoe", 1) for n, c in CASES.items() if n != "bf16_tok"]  # (name, cfg, schedule, lanes)
    runs = [(n, c, s, l, "nccl") for n, c, s, l in runs]
    runs += [("bf16_p_" + sch, CASES["bf16_p"], sch, lanes, "nccl")
             for sch, lanes in (("flowmoe", 2), ("flowmoe_ar", 1), ("pipe_moe", 2), ("vanilla_ep", 1))]
    # peer-memory A2A (NVLink stores from our kernels) — same results as NCCL
    runs += [("c1_f32_p2p", CASES["c1_f32"], "flowmoe", 2, "p2p"),
             ("bf16_p_p2p", CASES["bf16_p"], "flowmoe", 2, "p2p"),
             ("bf16_p_p2p_vanilla", CASES["bf16_p"], "vanilla_ep", 1, "p2p"),
             ("bf16_tok_nccl", CASES["bf16_tok"], "flowmoe", 1, "nccl"),
             ("bf16_tok_p2p", CASES["bf16_tok"], "flowmoe", 4, "p2p")]
    for name, base, schedule, lanes, a2a in runs:
        cfg = base.replace(P=P)
        obj = [fm.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        rep = gen_replicated(cfg)
        wks = [gen_worker(cfg, p) for p in range(P)]
        # tiny S_p so the all-reduce is cut into many chunks incl. a remainder
        g = run_block_gpu(cfg, rep, wks[rank], P=P, rank=rank, uid=obj[0], device=dev.index,
                          chunk_bytes=4096 + 16, schedule=schedule, compute_streams=lanes, a2a_impl=a2a,
                          repeat=(2 if a2a == "p2p" else 1))
        ocfg = cfg.replace(R=1) if schedule == "vanilla_ep" else cfg
        ys, dxs, gflat, eg, st = oracle_block(ocfg, rep, wks)
        El = cfg.E // P
        ref_e = expert_grads(eg, rank * El, (rank + 1) * El)
        r = {"y": rel(g["y"], ys[rank]), "dx": rel(g["dx"], dxs[rank]),
             "grad_flat": rel(g["grad_flat"], gflat)}
        for n in ("dw1", "db1", "dw2", "db2"):
            r[n] = rel(g[n], ref_e[n])
        ro = st.route[rank]
        r["routing_exact"] = bool(np.array_equal(g["idx"], ro.idx) and
                                  np.array_equal(g["pos"], np.where(ro.kept, ro.pos, -1)) and
                                  np.array_equal(g["counts"], ro.counts))
        results[name] = r
    # 3-block stack: per-block calls (forced routing) vs the oracle chain over P workers,
    # and the stack API (lanes forked once) vs per-block calls bit for bit
    L = 3
    for name, base, a2a in (("stack_f32", CASES["c1_f32"].replace(R=4, causal=1, residual=1), "nccl"),
                            ("stack_bf16_p2p", CASES["bf16_p"], "p2p"),
                            ("stack_bf16_nccl", CASES["bf16_p"], "nccl")):
        cfg = base.replace(P=P)
        reps = [gen_replicated(cfg, block=l) for l in range(L)]
        wks = [gen_worker(cfg, p) for p in range(P)]
        forced = [[gen_worker(cfg, p, block=l)["forced_idx"] for p in range(P)] for l in range(L)]
        runs_api = {}
        for api, fr in (("per_block", True), ("per_block_free", False), ("stack", False)):
            obj = [fm.get_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            wk = dict(wks[rank])
            wk["forced"] = [forced[l][rank] for l in range(L)] if fr else None
            runs_api[api] = run_stack_gpu(cfg, reps, wk, compute_streams=cfg.R, device=dev.index,
                                          api="stack" if api == "stack" else "per_block", P=P, rank=rank,
                                          uid=obj[0], a2a_impl=a2a, chunk_bytes=4096 + 16,
                                          graph=(api == "stack"))
        # per-block parity: the oracle's P workers run block l on every rank's GPU input
        # to that block (single-block tolerance, no compounding through the chain)
        mine = {n: runs_api["per_block"][n] for n in ("xs", "dxs", "grad_flat", "dw1")}
        allg = [None] * P
        dist.all_gather_object(allg, mine)
        r = chain_per_block_errors(cfg, reps, [[forced[l][p] for l in range(L)] for p in range(P)],
                                   [w["dy"] for w in wks], allg, rank=rank, P=P)
        a, b = runs_api["stack"], runs_api["per_block_free"]
        r["stack_bitwise"] = bool(all(np.array_equal(a[n], b[n]) for n in ("y", "dx")) and all(
            np.array_equal(a[n][l], b[n][l]) for n in ("grad_flat", "dw1") for l in range(L)))
        results[name] = r
    # schedule properties on the measured timeline of a real P-rank stack iteration
    # (SURVEY §8(c.3)): orders, 6a-6e, FIFO per stream, AR order and the priority rule
    from paper_2510_00207_b200.schedule import check_schedule, violations
    cfg = BlockConfig(T=1024, seq_len=256, M=512, n_heads=4, E=8, top_k=2, d_ffn=1024, R=4,
                      capacity_factor=1.0, causal=1, residual=1, dtype="bf16", P=P)
    for a2a in ("p2p", "nccl"):
        L = 3
        reps = [gen_replicated(cfg, block=l) for l in range(L)]
        obj = [fm.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        wk = dict(gen_worker(cfg, rank), forced=None)
        g = run_stack_gpu(cfg, reps, wk, compute_streams=cfg.R, device=dev.index, api="stack", P=P, rank=rank,
                          uid=obj[0], a2a_impl=a2a, chunk_bytes=256 << 10, tasklog=True)
        res = check_schedule(g["log"], L, cfg.R, P)
        v = violations(res)
        results[f"sched_{a2a}"] = {"violations": {k: len(x) for k, x in v.items()},
                                   "examples": {k: [list(map(str, e)) for e in x[:6]] for k, x in v.items()},
                                   "checked": res["checked"], "priority": res["priority_stats"]}
    out = [None] * P
    dist.all_gather_object(out, results)
    if rank == 0:
        print("MP_RESULTS " + json.dumps(out), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
