"""Tune the AR chunk size S_p on real iterations (FlowMoE §4.1, Appendix D).

Runs under torchrun (one rank per GPU).  The objective F(S_p) is the mean device
time of `--iters` iterations of the L-block stack with the AR cut at S_p (each
candidate re-captures the CUDA graph).  Rank 0 drives paper_2510_00207_b200.bo
(BO: 1 random + 7 EI samples; grid: 8 equal parts; random: 8 draws) and broadcasts
each candidate.  Also sweeps a fixed ladder (0.5..8 MiB + whole tensor, the
paper's Table Sp_sensitivity ladder) for the Theorem 2 trade-off.  Prints JSON.

  python -m torch.distributed.run --nproc-per-node 2 tools/tune_sp.py --config c4
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--layers", type=int, default=0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--compute-streams", type=int, default=-1)
    ap.add_argument("--out", default="")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    import paper_2510_00207_b200 as fm
    from paper_2510_00207_b200 import bo
    from synth import PRESETS, gen_device_block, gen_device_worker
    import bench

    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    obj = [fm.get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    cfg = PRESETS[args.config].replace(P=world)
    L = args.layers or bench.LAYERS[args.config]
    lanes = cfg.R if args.compute_streams < 0 else args.compute_streams
    ctx = fm.FlowMoE(fm.BlockShape(B=cfg.T, seq_len=cfg.seq_len, M=cfg.M, n_heads=cfg.n_heads, E=cfg.E,
                                   top_k=cfg.top_k, d_ffn=cfg.d_ffn, R=cfg.R,
                                   capacity_factor=cfg.capacity_factor, causal=cfg.causal,
                                   residual=cfg.residual, dtype=cfg.dtype, world_size=world, rank=rank,
                                   grad_mode="overwrite", compute_streams=lanes), local, obj[0])
    blocks = []
    for l in range(L):
        w = gen_device_block(cfg, rank, world, l, dev)
        f32 = dict(device=dev, dtype=torch.float32)
        El = cfg.E // world
        g = {"grad_flat": torch.zeros(ctx.grad_flat_count, **f32),
             "dw1": torch.zeros(El, cfg.M, cfg.d_ffn, **f32), "db1": torch.zeros(El, cfg.d_ffn, **f32),
             "dw2": torch.zeros(El, cfg.d_ffn, cfg.M, **f32), "db2": torch.zeros(El, cfg.M, **f32)}
        blocks.append(dict(w=w, g=g, saved=torch.empty(ctx.saved_bytes, dtype=torch.uint8, device=dev),
                           params=fm.Params(*[w[n].data_ptr() for n in ("wqkv", "wo", "wg", "w1", "b1", "w2", "b2")]),
                           grads=fm.Grads(*[g[n].data_ptr() for n in ("grad_flat", "dw1", "db1", "dw2", "db2")])))
    x0, dy_top = gen_device_worker(cfg, rank, dev)
    xs = [x0] + [torch.empty_like(x0) for _ in range(L)]
    dxs = [torch.empty_like(x0) for _ in range(L)]

    def iteration(s, sp):
        for l in range(L):
            ctx.block_fwd(blocks[l]["params"], xs[l], xs[l + 1], blocks[l]["saved"], s)
        tickets, gin = [], dy_top
        for l in reversed(range(L)):
            tickets.append(ctx.block_bwd(blocks[l]["params"], xs[l], blocks[l]["saved"], gin, dxs[l],
                                         blocks[l]["grads"], sp, s))
            gin = dxs[l]
        for t in tickets:
            ctx.allreduce_wait(t, s)

    ar_bytes = 4 * ctx.grad_flat_count
    cache = {}

    def measure(sp_bytes: float) -> float:
        sp = int(max(16, min(ar_bytes, round(sp_bytes / 16) * 16)))
        if sp in cache:
            return cache[sp]
        stream = torch.cuda.current_stream()
        iteration(stream, sp)  # warm
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap, capture_error_mode="thread_local"):
            iteration(torch.cuda.current_stream(), sp)
        for _ in range(3):
            graph.replay()
        dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.iters):
            graph.replay()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / args.iters], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        del graph
        torch.cuda.synchronize()
        cache[sp] = float(t.item())
        return cache[sp]

    def driven(fn):
        """Rank 0 runs the tuner; every objective evaluation is broadcast so all ranks
        measure the same S_p (collective NCCL ops must match)."""
        if rank == 0:
            def obj_fn(v):
                dist.broadcast_object_list([v], src=0)
                return measure(v)
            res = fn(obj_fn)
            dist.broadcast_object_list([None], src=0)
            return res
        while True:
            box = [None]
            dist.broadcast_object_list(box, src=0)
            if box[0] is None:
                return None
            measure(box[0])

    MiB = 1 << 20
    out = {"config": args.config, "n_gpus": world, "layers": L, "ar_bytes_per_block": ar_bytes,
           "iters_per_sample": args.iters}
    ladder = [MiB // 2, MiB, 2 * MiB, 4 * MiB, 8 * MiB, ar_bytes]
    out["ladder_ms"] = driven(lambda f: {str(v): f(v) for v in ladder})
    out["bo"] = driven(lambda f: bo.bo_tune(f, 0.0, ar_bytes, budget=8, seed=0, quantum=16, xi_relative=True).__dict__)
    out["grid"] = driven(lambda f: bo.grid_tune(f, 0.0, ar_bytes, points=8, quantum=16).__dict__)
    out["random"] = driven(lambda f: bo.random_tune(f, 0.0, ar_bytes, draws=8, seed=1, quantum=16).__dict__)
    if rank == 0:
        line = json.dumps(out)
        print(line, flush=True)
        if args.out:
            open(args.out, "w").write(line + "\n")
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
