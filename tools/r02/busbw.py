"""NVLink bus bandwidth of the two exchanges, nccl-tests style, at N ranks (torchrun):
  - the chunked all-reduce of the replicated grads through the library's AR communicator
    (flowmoe_allreduce_submit: ncclAllReduce sum fp32, maxCTAs-capped) and, for reference,
    torch.distributed.all_reduce on the default NCCL communicator;
    busBW = bytes * 2(P-1)/P / t
  - one A2A exchange (dispatch D_r of one chunk) through NCCL send/recv groups and through
    the peer-memory kernel (flowmoe_test.h flowmoe_test_exchange), at the dsv2s / c4 / c3
    / c2 chunk shapes; busBW = E*C*M*2 * (P-1)/P / t (bytes leaving each rank).
Each point: barrier, CUDA-event time of `iters` back-to-back calls, max over ranks.
Rank 0 prints one JSON line per point and writes profiles/r02/busbw_n{P}.md.
  python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 tools/r02/busbw.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_2510_00207_b200 as fm  # noqa: E402
from synth import PRESETS  # noqa: E402


def timed(fn, iters, dev):
    dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn(iters)
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()) * 1e-3  # seconds per call


def main():
    rank, P = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    dev = torch.device("cuda", int(os.environ["LOCAL_RANK"]))
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    rows = []
    s = torch.cuda.current_stream()

    def uid():
        obj = [fm.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    # ---- all-reduce
    base = PRESETS["c2"].replace(P=P)
    shape = fm.BlockShape(B=base.T, seq_len=base.seq_len, M=base.M, n_heads=base.n_heads, E=base.E, top_k=base.top_k,
                          d_ffn=base.d_ffn, R=base.R, world_size=P, rank=rank)
    ctx = fm.FlowMoE(shape, dev.index, uid())
    for mib in (1, 4, 16, 64, 256):
        n = mib * (1 << 20) // 4
        buf = torch.ones(n, device=dev)

        def lib_ar(iters):
            for _ in range(iters):
                ctx.allreduce_wait(ctx.allreduce_submit(buf, n, n * 4), s)

        def torch_ar(iters):
            for _ in range(iters):
                dist.all_reduce(buf)
        for name, fn in (("allreduce (library AR comm, maxCTAs cap)", lib_ar), ("allreduce (torch.distributed)", torch_ar)):
            fn(3)
            t = timed(fn, 20, dev)
            rows.append({"op": name, "bytes": n * 4, "us": t * 1e6, "busbw_gbs": n * 4 * 2 * (P - 1) / P / t / 1e9})
    ctx.close()
    # ---- A2A exchange of one chunk
    for cname in ("dsv2s", "c4", "c3", "c2"):
        cfg = PRESETS[cname].replace(P=P)
        if cfg.E % P:
            continue
        for impl in ("nccl", "p2p"):
            shape = fm.BlockShape(B=cfg.T, seq_len=cfg.seq_len, M=cfg.M, n_heads=cfg.n_heads, E=cfg.E,
                                  top_k=cfg.top_k, d_ffn=cfg.d_ffn, R=cfg.R, capacity_factor=cfg.capacity_factor,
                                  causal=cfg.causal, residual=cfg.residual, world_size=P, rank=rank, a2a_impl=impl)
            ctx = fm.FlowMoE(shape, dev.index, uid())
            saved = torch.zeros(ctx.saved_bytes, dtype=torch.uint8, device=dev)
            ctx.register_saved(saved)
            import math
            C = math.ceil(cfg.capacity_factor * cfg.top_k * (cfg.T // cfg.R) / cfg.E)
            nbytes = cfg.E * C * cfg.M * 2

            def ex(iters):
                ctx.test_exchange(saved, 0, 0, iters, s)
            ex(3)
            t = timed(ex, 20, dev)
            rows.append({"op": f"A2A dispatch, {cname} chunk ({impl})", "bytes": nbytes, "us": t * 1e6,
                         "busbw_gbs": nbytes * (P - 1) / P / t / 1e9})
            ctx.close()
            del saved
    if rank == 0:
        for r in rows:
            print(json.dumps(dict(r, n_gpus=P)), flush=True)
        os.makedirs(os.path.join(ROOT, "profiles", "r02"), exist_ok=True)
        with open(os.path.join(ROOT, "profiles", "r02", f"busbw_n{P}.md"), "w") as f:
            f.write(f"# NVLink bus bandwidth at {P} B200 (tools/r02/busbw.py; max over ranks of 20 calls)\n\n")
            f.write("busBW: all-reduce bytes*2(P-1)/P/t, A2A bytes*(P-1)/P/t; nominal 900 GB/s per direction, "
                    "measured references 725 GB/s (8-rank AR) and 770 GB/s (peer copy), B200_PROFILING.md\n\n")
            f.write("| op | bytes per rank | µs per call | busBW GB/s | of 900 |\n|---|---|---|---|---|\n")
            for r in rows:
                f.write(f"| {r['op']} | {r['bytes'] / 2**20:.2f} MiB | {r['us']:.1f} | {r['busbw_gbs']:.0f} | "
                        f"{r['busbw_gbs'] / 900:.2f} |\n")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
