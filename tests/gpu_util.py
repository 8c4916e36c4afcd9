"""Helpers shared by the GPU parity tests: run one FlowMoE block through the
C ABI on seeded synth inputs and return everything as fp64 numpy arrays."""
from __future__ import annotations

import numpy as np

import paper_2510_00207_b200 as fm
from synth import BlockConfig


def rel(g: np.ndarray, r: np.ndarray) -> float:
    """max |g - r| / max |r| (the north_star metric, per tensor)."""
    den = float(np.max(np.abs(r)))
    return float(np.max(np.abs(g - r))) / (den if den > 0 else 1.0)


def shape_of(cfg: BlockConfig, P: int, rank: int, grad_mode: str = "accumulate",
             compute_streams: int = 1, schedule: str = "flowmoe", a2a_impl: str = "nccl") -> fm.BlockShape:
    return fm.BlockShape(B=cfg.T, seq_len=cfg.seq_len, M=cfg.M, n_heads=cfg.n_heads, E=cfg.E,
                         top_k=cfg.top_k, d_ffn=cfg.d_ffn, R=cfg.R,
                         capacity_factor=cfg.capacity_factor, causal=cfg.causal,
                         residual=cfg.residual, dtype=cfg.dtype, world_size=P, rank=rank,
                         grad_mode=grad_mode, compute_streams=compute_streams, schedule=schedule,
                         a2a_impl=a2a_impl)


def run_block_gpu(cfg: BlockConfig, rep: dict, wk: dict, *, P: int = 1, rank: int = 0,
                  forced: bool = True, chunk_bytes: int = 1 << 20, uid: bytes | None = None,
                  device: int = 0, grad_mode: str = "accumulate", repeat_bwd: int = 1,
                  grad_fill: float = 0.0, compute_streams: int = 1,
                  schedule: str = "flowmoe", a2a_impl: str = "nccl", repeat: int = 1) -> dict:
    import torch
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    ctx = fm.FlowMoE(shape_of(cfg, P, rank, grad_mode, compute_streams, schedule, a2a_impl), device, uid)
    bt = fm.BlockTensors(rep, cfg.dtype, rank, P, dev)
    if grad_fill:
        for v in bt.g.values():
            v.fill_(grad_fill)
    x = fm.to_device(wk["x"], cfg.dtype, dev)
    dy = fm.to_device(wk["dy"], cfg.dtype, dev)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    saved = torch.empty(ctx.saved_bytes, dtype=torch.uint8, device=dev)
    fidx = None
    if forced:
        fidx = torch.from_numpy(np.ascontiguousarray(wk["forced_idx"], dtype=np.int32)).to(dev)
        ctx.set_forced_routing(fidx)
    s = torch.cuda.current_stream()
    for it in range(repeat):  # repeat > 1 re-runs the iteration (A2A counters/epochs advance)
        if it:
            for v in bt.g.values():
                v.zero_()
        ctx.block_fwd(bt.params, x, y, saved, s)
        for _ in range(repeat_bwd):
            t = ctx.block_bwd(bt.params, x, saved, dy, dx, bt.grads, chunk_bytes, s)
            ctx.allreduce_wait(t, s)
    torch.cuda.synchronize()
    off = ctx.routing_offsets()
    T, E, k, R = cfg.T, cfg.E, cfg.top_k, (1 if schedule == "vanilla_ep" else cfg.R)

    def view(o, n, dt):
        nbytes = n * 4
        return saved[o:o + nbytes].view(dt).cpu().numpy().copy()

    out = {
        "y": fm.to_host_f64(y), "dx": fm.to_host_f64(dx),
        "grad_flat": bt.g["grad_flat"].cpu().numpy().astype(np.float64),
        "dw1": bt.g["dw1"].cpu().numpy().astype(np.float64),
        "db1": bt.g["db1"].cpu().numpy().astype(np.float64),
        "dw2": bt.g["dw2"].cpu().numpy().astype(np.float64),
        "db2": bt.g["db2"].cpu().numpy().astype(np.float64),
        "logits": view(off["logits"], T * E, torch.float32).reshape(T, E),
        "idx": view(off["idx"], T * k, torch.int32).reshape(T, k),
        "w": view(off["w"], T * k, torch.float32).reshape(T, k),
        "pos": view(off["pos"], T * k, torch.int32).reshape(T, k),
        "counts": view(off["counts"], R * E, torch.int32).reshape(R, E),
    }
    ctx.close()
    return out


def oracle_block(cfg: BlockConfig, rep: dict, wks: list[dict], forced: bool = True):
    """Oracle fwd+bwd over len(wks) workers (fp64)."""
    import oracle as o
    xs = [w["x"] for w in wks]
    dys = [w["dy"] for w in wks]
    fidx = [w["forced_idx"] for w in wks] if forced else None
    ys, st = o.block_forward(cfg, rep, xs, fidx)
    dxs, gflat, eg = o.block_backward(cfg, rep, st, dys)
    return ys, dxs, gflat, eg, st


def expert_grads(eg: dict, lo: int, hi: int):
    return {name: np.stack([eg[e][i] for e in range(lo, hi)])
            for i, name in enumerate(("dw1", "db1", "dw2", "db2"))}


class HostGate:
    """Holds a stream at a device-side wait (cuStreamWaitValue32, a stream memory operation —
    no kernel spins) on a device flag until release() writes the flag from another stream:
    everything enqueued behind the gate is queued before the GPU starts any of it, so measured
    task timelines carry no host-enqueue gaps (the schedule-property checks compare task start
    times with their ready times)."""

    def __init__(self, stream):
        import ctypes

        import torch
        self.flag = torch.zeros(1, dtype=torch.int32, device=stream.device)
        torch.cuda.synchronize()
        self.cu = ctypes.CDLL("libcuda.so.1")
        self.cu.cuStreamWaitValue32_v2.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
        self.cu.cuStreamWriteValue32_v2.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint]
        rc = self.cu.cuStreamWaitValue32_v2(ctypes.c_void_p(stream.cuda_stream), ctypes.c_uint64(self.flag.data_ptr()),
                                         1, 0)  # CU_STREAM_WAIT_VALUE_GEQ
        assert rc == 0, f"cuStreamWaitValue32: CUresult {rc}"
        self.side = torch.cuda.Stream(device=stream.device)

    def release(self):
        import ctypes
        rc = self.cu.cuStreamWriteValue32_v2(ctypes.c_void_p(self.side.cuda_stream), ctypes.c_uint64(self.flag.data_ptr()),
                                          1, 0)
        assert rc == 0, f"cuStreamWriteValue32: CUresult {rc}"


def run_stack_gpu(cfg: BlockConfig, reps: list, wk: dict, *, compute_streams: int = 1,
                  schedule: str = "flowmoe", graph: bool = False, device: int = 0,
                  api: str = "per_block", P: int = 1, rank: int = 0, uid: bytes | None = None,
                  a2a_impl: str = "nccl", chunk_bytes: int = 1 << 20, tasklog: bool = False) -> dict:
    """L = len(reps) blocks chained through the C ABI on one rank (forced routing per
    block from wk['forced'][l], or the gate's own routing when wk['forced'] is None):
    forward x -> y_L, backward from wk['dy'] to dx_0.  api='stack' drives the same
    iteration through flowmoe_stack_fwd / flowmoe_stack_bwd."""
    import torch
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    ctx = fm.FlowMoE(shape_of(cfg, P, rank, "overwrite", compute_streams, schedule, a2a_impl), device, uid)
    L = len(reps)
    bts = [fm.BlockTensors(r, cfg.dtype, rank, P, dev) for r in reps]
    xs = [fm.to_device(wk["x"], cfg.dtype, dev)] + [None] * L
    for l in range(L):
        xs[l + 1] = torch.empty_like(xs[0])
    dxs = [torch.empty_like(xs[0]) for _ in range(L)]
    dy = fm.to_device(wk["dy"], cfg.dtype, dev)
    saved = [torch.empty(ctx.saved_bytes, dtype=torch.uint8, device=dev) for _ in range(L)]
    forced = None if wk.get("forced") is None else \
        [torch.from_numpy(np.ascontiguousarray(f, dtype=np.int32)).to(dev) for f in wk["forced"]]
    assert api == "per_block" or forced is None, "stack API runs the gate's own routing"

    def iteration(s):
        if api == "stack":
            ctx.stack_fwd([b.params for b in bts], xs[0], xs[1:], saved, s)
            for t in ctx.stack_bwd([b.params for b in bts], xs[0], xs[1:], saved, dy, dxs,
                                   [b.grads for b in bts], chunk_bytes, s):
                ctx.allreduce_wait(t, s)
            return
        for l in range(L):
            if forced is not None:
                ctx.set_forced_routing(forced[l])
            ctx.block_fwd(bts[l].params, xs[l], xs[l + 1], saved[l], s)
        g, tickets = dy, []
        for l in reversed(range(L)):
            tickets.append(ctx.block_bwd(bts[l].params, xs[l], saved[l], g, dxs[l], bts[l].grads, chunk_bytes, s))
            g = dxs[l]
        for t in tickets:
            ctx.allreduce_wait(t, s)

    s = torch.cuda.current_stream()
    iteration(s)
    log = None
    if tasklog:  # a second eager iteration with the task log on (schedule properties), fully
        torch.cuda.synchronize()  # enqueued behind a host gate before the GPU runs any of it
        ctx.tasklog_begin()
        gate = HostGate(s)
        iteration(s)
        gate.release()
        log = ctx.tasklog_end()
    if graph:  # capture the same iteration and replay it twice (overwrite grads -> same values)
        for bt in bts:
            for v in bt.g.values():
                v.fill_(7.0)
        gr = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(s)
        with torch.cuda.graph(gr, stream=cap, capture_error_mode="thread_local"):
            iteration(torch.cuda.current_stream())
        gr.replay()
        gr.replay()
    torch.cuda.synchronize()
    out = {"y": fm.to_host_f64(xs[L]), "dx": fm.to_host_f64(dxs[0]),
           "xs": [fm.to_host_f64(t) for t in xs], "dxs": [fm.to_host_f64(t) for t in dxs],
           "grad_flat": [bt.g["grad_flat"].cpu().numpy().astype(np.float64) for bt in bts],
           "dw1": [bt.g["dw1"].cpu().numpy().astype(np.float64) for bt in bts], "log": log}
    if graph:
        del gr
        torch.cuda.synchronize()
    ctx.close()
    return out


def chain_per_block_errors(cfg, reps, forced, dy_top, g, rank=0, P=1):
    """Per-block parity of an L-block chain: the oracle runs block l on the GPU's own input
    to that block (x_l, and for the backward the GPU's dx_{l+1}), so every block is held to
    the single-block tolerance (no compounding of bf16 rounding through the chain).  With
    P > 1 every worker's GPU inputs are needed: `g` is then the list of per-rank results."""
    import oracle as o
    gs = g if isinstance(g, list) else [g]
    L = len(reps)
    res = {}
    for l in range(L):
        xin = [gg["xs"][l] for gg in gs]
        ys, st = o.block_forward(cfg, reps[l], xin, [f[l] for f in forced] if forced else None)
        dyin = [(gg["dxs"][l + 1] if l + 1 < L else dy_top[q]) for q, gg in enumerate(gs)]
        dxl, gflat, eg = o.block_backward(cfg, reps[l], st, dyin)
        me = gs[rank] if len(gs) > 1 else gs[0]
        El = cfg.E // P
        res[f"y{l}"] = rel(me["xs"][l + 1], ys[rank])
        res[f"dx{l}"] = rel(me["dxs"][l], dxl[rank])
        res[f"grad_flat{l}"] = rel(me["grad_flat"][l], gflat)
        res[f"dw1_{l}"] = rel(me["dw1"][l], np.stack([eg[e][0] for e in range(rank * El, (rank + 1) * El)]))
    return res


def run_group_gpu(cfg: BlockConfig, rep: dict, wks: list, *, forced: bool = True, chunk_bytes: int = 4096 + 16,
                  compute_streams: int = 1, schedule: str = "flowmoe", repeat: int = 2, device: int = 0,
                  stack_reps: list | None = None) -> list:
    """P = len(wks) ranks of one block (or, with stack_reps, an L-block stack through the
    stack API) in the in-process simulated world on ONE GPU (flowmoe_create_local_group):
    the real peer-memory A2A send kernels move the blocks between the ranks' buffers and the
    all-reduce runs the S_p chunk loop.  Every rank is driven by its own host thread (the
    exchanges meet at host barriers; no kernel waits for another launch), the all-reduce
    waits run once every rank's backward is enqueued.  repeat > 1 re-runs the iteration.
    Returns per-rank results, incl. the A2A arrival counters."""
    import threading

    import torch
    P = len(wks)
    dev = torch.device("cuda", device)
    torch.cuda.set_device(dev)
    shape = shape_of(cfg, P, 0, "overwrite", compute_streams, schedule, "p2p")
    ctxs = fm.FlowMoE.local_group(shape, P, device)
    reps = stack_reps if stack_reps is not None else [rep]
    L = len(reps)
    bts = [[fm.BlockTensors(r, cfg.dtype, q, P, dev) for r in reps] for q in range(P)]
    xs = [[fm.to_device(wks[q]["x"], cfg.dtype, dev)] + [None] * L for q in range(P)]
    for q in range(P):
        for l in range(L):
            xs[q][l + 1] = torch.empty_like(xs[q][0])
    dxs = [[torch.empty_like(xs[q][0]) for _ in range(L)] for q in range(P)]
    dys = [fm.to_device(wks[q]["dy"], cfg.dtype, dev) for q in range(P)]
    saved = [[torch.empty(ctxs[q].saved_bytes, dtype=torch.uint8, device=dev) for _ in range(L)] for q in range(P)]
    for l in range(L):  # collective registration, same order on every rank
        for q in range(P):
            ctxs[q].register_saved(saved[q][l])
    fidx = None
    if forced:  # the same forced indices for every block of a stack
        fidx = [torch.from_numpy(np.ascontiguousarray(wks[q]["forced_idx"], dtype=np.int32)).to(dev)
                for q in range(P)]
        for q in range(P):
            ctxs[q].set_forced_routing(fidx[q])
    s = torch.cuda.current_stream()
    torch.cuda.synchronize()

    def rank_fwd_bwd(q, tickets):
        torch.cuda.set_device(dev)
        if stack_reps is not None:
            ctxs[q].stack_fwd([b.params for b in bts[q]], xs[q][0], xs[q][1:], saved[q], s)
            tickets[q] = ctxs[q].stack_bwd([b.params for b in bts[q]], xs[q][0], xs[q][1:], saved[q], dys[q],
                                           dxs[q], [b.grads for b in bts[q]], chunk_bytes, s)
        else:
            ctxs[q].block_fwd(bts[q][0].params, xs[q][0], xs[q][1], saved[q][0], s)
            tickets[q] = [ctxs[q].block_bwd(bts[q][0].params, xs[q][0], saved[q][0], dys[q], dxs[q][0],
                                            bts[q][0].grads, chunk_bytes, s)]

    for _ in range(repeat):
        tickets, errs = [None] * P, [None] * P

        def body(q):
            try:
                rank_fwd_bwd(q, tickets)
            except BaseException as e:  # re-raised below
                errs[q] = e
        th = [threading.Thread(target=body, args=(q,)) for q in range(P)]
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
    torch.cuda.synchronize()
    for c in ctxs:
        c.check_health()
    out = []
    T, E, k, R = cfg.T, cfg.E, cfg.top_k, cfg.R
    for q in range(P):
        off = ctxs[q].routing_offsets()

        def view(o, n, dt, q=q):
            return saved[q][0][o:o + n * 4].view(dt).cpu().numpy().copy()

        out.append({
            "y": fm.to_host_f64(xs[q][L]), "dx": fm.to_host_f64(dxs[q][0]),
            "xs": [fm.to_host_f64(t) for t in xs[q]], "dxs": [fm.to_host_f64(t) for t in dxs[q]],
            "grad_flat_l": [bt.g["grad_flat"].cpu().numpy().astype(np.float64) for bt in bts[q]],
            "dw1_l": [bt.g["dw1"].cpu().numpy().astype(np.float64) for bt in bts[q]],
            "grad_flat": bts[q][0].g["grad_flat"].cpu().numpy().astype(np.float64),
            **{n: bts[q][0].g[n].cpu().numpy().astype(np.float64) for n in ("dw1", "db1", "dw2", "db2")},
            "idx": view(off["idx"], T * k, torch.int32).reshape(T, k),
            "pos": view(off["pos"], T * k, torch.int32).reshape(T, k),
            "counts": view(off["counts"], R * E, torch.int32).reshape(R, E),
            "arrivals": ctxs[q].arrivals(),
        })
    for c in ctxs:
        c.close()
    return out
