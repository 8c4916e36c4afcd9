#!/usr/bin/env python
"""FlowMoE block-stack training-iteration benchmark (B200, sm_100a).

One step = one training iteration of an L-block transformer-MoE stack through
the C ABI (libflowmoe.so): flowmoe_stack_fwd over the L blocks, then
flowmoe_stack_bwd in reverse order (each block auto-submitting the chunked S_p
all-reduce of its MHA+gate grads), then flowmoe_allreduce_wait on every ticket (Alg. 1 lines 6-22, P:258-309;
the optimizer update, line 23, is excluded as in SURVEY.md §8(d)).  Weights and
inputs are synthetic (synth.gen_device_*), resident in HBM before the timed
region.  The iteration is captured once into a CUDA graph and replayed.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

N>1 is launched by torchrun (one rank per GPU, NCCL); weak scaling: T tokens per
rank fixed, E experts fixed, E/P local experts per rank.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MoE block iteration ms & tokens/s at 1/2/4/8 B200; exposed comm %"  # BASELINE.json metric
LAYERS = {"c1": 1, "c2": 12, "c3": 4, "c4": 4, "dsv2s": 4}   # Table 3 L for c2; §8(d) L in {1,4} else
# S_p defaults from BO on 2x B200 (profiles/r01/tune/): NCCL's per-call cost on NVLink puts the
# optimum at (or near) the whole per-block tensor; 0 = whole tensor
# S_p per config from the BO / grid tuning on B200 (profiles/r01/tune_n4/; 0 = whole tensor)
SP_DEFAULT = {"c1": 0, "c2": 0, "c3": 16 << 20, "c4": 96 << 20, "dsv2s": 0}
CONFIG_NAMES = {
    "c1": "configs[0] single fp32 MoE block (T=256, M=64, 4 heads, E=4 top-2, F=128, R=2)",
    "c2": "configs[1] GPT2-Tiny-MoE-shaped block stack (M=256, 4 heads, E=8 top-2, F=512, R=4, L=12)",
    "c3": "configs[2] BERT-Large-MoE-shaped (M=1024, 16 heads, E=16 top-2, F=2048, R=2)",
    "c4": "configs[3] LLaMA2-MoE-shaped (M=4096, 32 heads, E=16 top-2, F=16384, R=2)",
    "dsv2s": "configs[4] DeepSeek-V2-S-shaped (M=5120, 40 heads, E=16 top-8, F=1536, R=2)",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="flowmoe", choices=["flowmoe", "reference"])
    ap.add_argument("--config", default="dsv2s", choices=sorted(LAYERS),
                    help="workload (default: configs[4] DeepSeek-V2-S-shaped, the largest single-GPU config)")
    ap.add_argument("--layers", type=int, default=0, help="blocks in the stack (default per config)")
    ap.add_argument("--R", type=int, default=0, help="override pipelining degree")
    ap.add_argument("--chunk-bytes", type=int, default=0, help="S_p (default per config)")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--optimizer", default="", choices=["", "sgd", "adamw"],
                    help="include the parameter update (P:1173 placement: experts behind their wgrads, "
                         "replicated weights after their all-reduce); not part of the paper's metric")
    ap.add_argument("--per-block", action="store_true",
                    help="L block_fwd/block_bwd calls (lanes joined per block) instead of the stack API")
    ap.add_argument("--schedule", default="flowmoe",
                    choices=["flowmoe", "flowmoe_ar", "flowmoe_at", "pipe_moe", "vanilla_ep"],
                    help="scheduling policy (the paper's Table 6 ablation)")
    ap.add_argument("--a2a", default="p2p", choices=["nccl", "p2p"],
                    help="A2A: NCCL send/recv groups or peer-memory kernels over NVLink")
    ap.add_argument("--compute-streams", type=int, default=-1,
                    help="compute lanes (1 = paper's single compute stream; default R)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-json", default="", help="write the per-kernel table here")
    ap.add_argument("--trace-dir", default="/tmp", help="where the CUPTI chrome traces are written")
    ap.add_argument("--trace-iters", type=int, default=20,
                    help="CUDA-graph replays traced with CUPTI (timeline, exposed comm); 0 = off")
    return ap.parse_args()


def load_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0,
                "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while running."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = os.path.join("/tmp", f"flowmoe_clocks_{os.getpid()}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower().startswith("active")})
        under_load = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(under_load) if under_load else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()), default=None)}


def host_cpu():
    """os.cpu_count() and the CPU model (lscpu, else /proc/cpuinfo) of this host."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((l.split(":", 1)[1].strip() for l in out.splitlines() if l.startswith("Model name")), None)
    except Exception:
        pass
    if model is None:
        try:
            model = next((l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")),
                         None)
        except Exception:
            pass
    return {"cpu_count": os.cpu_count(), "model": model}


def oracle_sample(cfg):
    """The bounded oracle sample: ONE sequence (seq_len tokens) of one block, fwd + bwd at
    the workload's shapes, P = 1 (every expert local), R = 1.  Its tokens/s is the L-block
    iteration's: attention is per sequence and everything else is per token, so the work
    scales with tokens and blocks (t_iter = t_sample · (T / seq_len) · L)."""
    import oracle as o
    from synth import gen_replicated, gen_worker
    one = cfg.replace(P=1, T=cfg.seq_len, R=1)
    rep = gen_replicated(one)
    wk = gen_worker(one, 0)

    def step():
        ys, st = o.block_forward(one, rep, [wk["x"]])
        o.block_backward(one, rep, st, [wk["dy"]])
    return one, step


def cpu_oracle_baseline(cfg, L, budget_s=12.0):
    """Time the fp64 oracle (as it stands) on this host's cores, twice: single-threaded
    (BLAS threads = 1, the plain oracle) and with every core (BLAS threads = nproc).  Each
    timing repeats the bounded sample (oracle_sample) until ~budget_s / 2 have passed."""
    from threadpoolctl import threadpool_info, threadpool_limits
    one, step = oracle_sample(cfg)
    res = {}
    for label, limit in (("single_thread", 1), ("all_cores", os.cpu_count() or 1)):
        with threadpool_limits(limits=limit):
            threads = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
            n, t = 0, 0.0
            while t < budget_s / 2 or n == 0:
                t0 = time.perf_counter()
                step()
                t += time.perf_counter() - t0
                n += 1
        t_sample = t / n
        res[label] = {"value": one.T / (t_sample * L), "s_per_sample": t_sample, "samples": n, "cores": threads}
    best = res["all_cores"]
    return {"value": best["value"], "unit": "tokens/s", "cores": best["cores"], "kind": "oracle",
            "sample": f"1 sequence ({one.T} tokens) of 1 block fwd+bwd at the workload's shapes (P=1, fp64 numpy), "
                      f"scaled to the {L}-block iteration (tokens/s = tokens / (t_sample * {L}))",
            "single_thread": res["single_thread"], "all_cores": res["all_cores"], "host": host_cpu()}


def run_reference(args, cfg, L, rank, world):
    """--impl reference: the fp64 oracle on the host cores (rank 0 only; this tier has no
    reference code to install).  Each step is the bounded sample of the same workload
    (oracle_sample: one sequence through one block, fwd + bwd), timed whole; ms_per_step is
    that measured sample time and value the tokens/s it implies for the L-block iteration."""
    if rank != 0:
        return
    from threadpoolctl import threadpool_info
    cores = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    one, step = oracle_sample(cfg)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        step()
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    t_sample = statistics.mean(times)
    value = one.T / (t_sample * L) * world       # whole job (weak scaling: every rank has T tokens)
    sample = (f"per step: 1 sequence ({one.T} tokens) of 1 block fwd+bwd (fp64 oracle); value = the "
              f"{L}-block iteration's tokens/s implied by it (tokens / (t_step * {L}))")
    line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_sample * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": CONFIG_NAMES[args.config], "tokens_per_gpu": cfg.T,
                       "seq_len": cfg.seq_len, "M": cfg.M, "n_heads": cfg.n_heads, "E": cfg.E,
                       "top_k": cfg.top_k, "d_ffn": cfg.d_ffn, "R": cfg.R, "layers": L,
                       "capacity_factor": cfg.capacity_factor, "parallelism": f"ep{world}+dp{world}",
                       "runs": "rank 0 only, host cores (fp64 oracle)", "step": sample},
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": cores, "kind": "oracle",
                             "sample": sample, "host": host_cpu()},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    import faulthandler
    import signal
    faulthandler.register(signal.SIGTERM, all_threads=True, chain=True)  # a killed run says where it was
    from synth import PRESETS
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    L = args.layers or LAYERS[args.config]
    cfg = PRESETS[args.config]
    if args.R:
        cfg = cfg.replace(R=args.R)
    cfg = cfg.replace(P=world)
    if args.impl == "reference":
        run_reference(args, cfg, L, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2510_00207_b200 as fm
    from synth import gen_device_block, gen_device_worker

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [fm.get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    S_p = args.chunk_bytes or SP_DEFAULT[args.config]
    if S_p <= 0:  # whole per-block AR tensor in one chunk
        S_p = 4 * (4 * cfg.M * cfg.M + cfg.M * cfg.E)
    S_p = (S_p + 15) // 16 * 16
    if args.compute_streams < 0:
        args.compute_streams = cfg.R
    shape = fm.BlockShape(B=cfg.T, seq_len=cfg.seq_len, M=cfg.M, n_heads=cfg.n_heads, E=cfg.E,
                          top_k=cfg.top_k, d_ffn=cfg.d_ffn, R=cfg.R,
                          capacity_factor=cfg.capacity_factor, causal=cfg.causal,
                          residual=cfg.residual, dtype=cfg.dtype, world_size=world, rank=rank,
                          grad_mode="overwrite",  # fresh grads each iteration (zero_grad + backward)
                          compute_streams=args.compute_streams, schedule=args.schedule,
                          a2a_impl=args.a2a)
    ctx = fm.FlowMoE(shape, local, uid)

    # ---- resident synthetic state
    blocks = []
    for l in range(L):
        w = gen_device_block(cfg, rank, world, l, dev)
        f32 = dict(device=dev, dtype=torch.float32)
        El = cfg.E // world
        g = {"grad_flat": torch.zeros(ctx.grad_flat_count, **f32),
             "dw1": torch.zeros(El, cfg.M, cfg.d_ffn, **f32), "db1": torch.zeros(El, cfg.d_ffn, **f32),
             "dw2": torch.zeros(El, cfg.d_ffn, cfg.M, **f32), "db2": torch.zeros(El, cfg.M, **f32)}
        params = fm.Params(*[w[n].data_ptr() for n in ("wqkv", "wo", "wg", "w1", "b1", "w2", "b2")])
        grads = fm.Grads(*[g[n].data_ptr() for n in ("grad_flat", "dw1", "db1", "dw2", "db2")])
        blocks.append(dict(w=w, g=g, params=params, grads=grads,
                           saved=torch.empty(ctx.saved_bytes, dtype=torch.uint8, device=dev)))
    x0, dy_top = gen_device_worker(cfg, rank, dev)
    xs = [x0] + [torch.empty_like(x0) for _ in range(L)]
    dxs = [torch.empty_like(x0) for _ in range(L)]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2

    plist = [b["params"] for b in blocks]
    glist = [b["grads"] for b in blocks]
    slist = [b["saved"] for b in blocks]

    opt = None
    if args.optimizer:  # fp32 master weights + optimizer state for every parameter
        import ctypes
        opt = fm.Optimizer.make(args.optimizer, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
        enames, rnames = ("w1", "b1", "w2", "b2"), ("wqkv", "wo", "wg")
        for b in blocks:
            b["master"] = {n: b["w"][n].float().clone() for n in enames + rnames}
            b["s1"] = {n: torch.zeros_like(b["master"][n]) for n in b["master"]}
            b["s2"] = {n: torch.zeros_like(b["master"][n]) for n in b["master"]} if args.optimizer == "adamw" else \
                {n: None for n in b["master"]}
            vp4 = ctypes.c_void_p * 4
            b["eopt"] = fm.ExpertOpt(vp4(*[b["master"][n].data_ptr() for n in enames]),
                                     vp4(*[b["s1"][n].data_ptr() for n in enames]),
                                     vp4(*[(b["s2"][n].data_ptr() if b["s2"][n] is not None else 0) for n in enames]),
                                     vp4(*[b["w"][n].data_ptr() for n in enames]))
            gf, M_, E_ = b["g"]["grad_flat"], cfg.M, cfg.E
            b["rgrad"] = {"wqkv": gf[:3 * M_ * M_], "wo": gf[3 * M_ * M_:4 * M_ * M_], "wg": gf[4 * M_ * M_:]}

    def replicated_update(stream):
        for b in blocks:
            for n in ("wqkv", "wo", "wg"):
                ctx.optimizer_step(opt, 1, b["master"][n], b["s1"][n], b["s2"][n], b["rgrad"][n], b["w"][n], stream)

    def iteration(stream):
        if not args.per_block:  # lanes forked once per direction, chunk r chains across blocks
            ctx.stack_fwd(plist, x0, xs[1:], slist, stream)
            tickets = ctx.stack_bwd(plist, x0, xs[1:], slist, dy_top, dxs, glist, S_p, stream)
            if opt is not None:
                tickets += [ctx.expert_update(opt, 1, b["eopt"], b["grads"]) for b in blocks]
            for t in tickets:
                ctx.allreduce_wait(t, stream)
            if opt is not None:
                replicated_update(stream)
            return
        for l in range(L):  # Eq.(3)/(4) order, block after block
            ctx.block_fwd(blocks[l]["params"], xs[l], xs[l + 1], blocks[l]["saved"], stream)
        tickets = []
        g_in = dy_top
        for l in reversed(range(L)):  # Eq.(5)/(6): blocks L..1, AR of block l under block l-1
            tickets.append(ctx.block_bwd(blocks[l]["params"], xs[l], blocks[l]["saved"], g_in, dxs[l],
                                         blocks[l]["grads"], S_p, stream))
            if opt is not None:  # block l's experts update as soon as their grads are final
                tickets.append(ctx.expert_update(opt, 1, blocks[l]["eopt"], blocks[l]["grads"]))
            g_in = dxs[l]
        for t in tickets:  # Alg. 1 line 22: wait for all all-reduce before the update
            ctx.allreduce_wait(t, stream)
        if opt is not None:
            replicated_update(stream)

    stream = torch.cuda.current_stream()
    # warm-up (eager) + launch count of one iteration
    n0 = fm.kernel_launches()
    iteration(stream)
    launches_per_step = fm.kernel_launches() - n0
    for _ in range(max(0, args.warmup - 1)):
        iteration(stream)
    torch.cuda.synchronize()

    # per-kernel live timing (eager iteration, CUDA events on each kernel's own stream)
    ctx.profile_begin()
    for _ in range(2):
        iteration(stream)
    prof = ctx.profile_end()
    for p in prof:
        p["launches"] //= 2
        p["ms"] /= 2
        p["flops"] /= 2
        p["bytes"] /= 2

    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        cap.wait_stream(stream)
        with torch.cuda.graph(graph, stream=cap, capture_error_mode="thread_local"):
            iteration(torch.cuda.current_stream())
        run = graph.replay
    else:
        run = lambda: iteration(stream)  # noqa: E731
    for _ in range(args.warmup):
        run()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps outside the events
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        time.sleep(0.3)
        for i in range(args.steps):
            flush.zero_()
            starts[i].record(stream)
            run()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = statistics.mean(s.elapsed_time(e) for s, e in zip(starts, ends))
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())

    # ---- e2e: every step copies its inputs host->device from pinned memory and reads its
    # result (dx) back, as a training loop would, pipelined: a copy stream uploads step
    # i+1's x / dy into a staging buffer and downloads step i-1's dx while step i runs; the
    # compute stream only pays two device-side copies in and one out per step.  The timed
    # region runs from the first upload to the last download.
    K2 = min(args.steps, 20)
    x_h = x0.cpu().pin_memory()
    dy_h = dy_top.cpu().pin_memory()
    dx_h = [torch.empty_like(dxs[0], device="cpu").pin_memory() for _ in range(2)]
    cs = torch.cuda.Stream(device=dev)
    xst = [torch.empty_like(xs[0]) for _ in range(2)]
    dyst = [torch.empty_like(dy_top) for _ in range(2)]
    dxst = [torch.empty_like(dxs[0]) for _ in range(2)]
    ev = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
    up_done, consumed, dx_ready, down_done = ev(), ev(), ev(), ev()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    cs.wait_stream(stream)

    def upload(b, i):
        with torch.cuda.stream(cs):
            if i >= 2:  # staging buffer b was last read by step i-2's device copy
                cs.wait_event(consumed[b])
            xst[b].copy_(x_h, non_blocking=True)
            dyst[b].copy_(dy_h, non_blocking=True)
            up_done[b].record(cs)

    upload(0, 0)
    for i in range(K2):
        b = i % 2
        if i + 1 < K2:
            upload(1 - b, i + 1)
        stream.wait_event(up_done[b])
        xs[0].copy_(xst[b])
        dy_top.copy_(dyst[b])
        consumed[b].record(stream)
        run()
        if i >= 2:  # dx staging buffer b was last drained by step i-2's download
            stream.wait_event(down_done[b])
        dxst[b].copy_(dxs[0])
        dx_ready[b].record(stream)
        with torch.cuda.stream(cs):
            cs.wait_event(dx_ready[b])
            dx_h[b].copy_(dxst[b], non_blocking=True)
            down_done[b].record(cs)
    stream.wait_stream(cs)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = torch.tensor([e0.elapsed_time(e1) / K2], device=dev)
    if world > 1:
        dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
    e2e_ms = float(e2e_ms.item())

    # ---- CUPTI timeline of graph replays: steady-state kernel times, idle, exposed comm
    tl = None
    tl_nopdl = None
    # bytes one exchange moves over NVLink (send side): E·C·M·es·(P-1)/P, C per chunk
    import math
    C_ = cfg.T // cfg.R if cfg.capacity_factor == 0 else \
        math.ceil(float(cfg.capacity_factor) * cfg.top_k * (cfg.T // cfg.R) / cfg.E)
    a2a_bytes = cfg.E * C_ * cfg.M * (2 if cfg.dtype == "bf16" else 4) * (world - 1) / world
    if args.trace_iters > 0:
        from paper_2510_00207_b200.timeline import trace_replays
        try:
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            tl = trace_replays(run, args.trace_iters, os.path.join(args.trace_dir, f"flowmoe_trace_{args.config}_n{world}_r{rank}.json"),
                               trim=max(0, min(3, (args.trace_iters - 2) // 4)),
                               sync=(dist.barrier if world > 1 else None),
                               a2a_bytes=a2a_bytes)
        except Exception as e:  # the timeline is diagnostics, never the measurement
            tl = {"error": repr(e)}
        # Kernel execution intervals for the roofline (N = 1): with programmatic dependent
        # launch a kernel is pre-launched and its CUPTI interval includes the wait for its
        # predecessor, so the same iteration is captured once more with PDL off and traced;
        # its group intervals are the kernels' execution (the other lane still contends).
        if world == 1 and not args.no_graph:
            try:
                ctx.debug_set(4, 0)
                graph2 = torch.cuda.CUDAGraph()
                cap2 = torch.cuda.Stream()
                cap2.wait_stream(stream)
                with torch.cuda.graph(graph2, stream=cap2, capture_error_mode="thread_local"):
                    iteration(torch.cuda.current_stream())
                ctx.debug_set(4, 1)
                for _ in range(3):
                    graph2.replay()
                torch.cuda.synchronize()
                tl_nopdl = trace_replays(graph2.replay, args.trace_iters,
                                         os.path.join(args.trace_dir, f"flowmoe_trace_{args.config}_n1_nopdl.json"),
                                         trim=max(0, min(3, (args.trace_iters - 2) // 4)), a2a_bytes=a2a_bytes)
                del graph2
            except Exception as e:
                ctx.debug_set(4, 1)
                tl_nopdl = {"error": repr(e)}
        if world > 1:
            allt = [None] * world
            dist.all_gather_object(allt, tl)
            tl = {"per_rank": allt}

    if rank == 0:
        peaks, peak_src = load_peaks()
        tokens = cfg.T * world
        compute = [p for p in prof if not p["name"].startswith(("a2a", "allreduce"))]
        total_ms = sum(p["ms"] for p in compute)
        tc_attn = cfg.dtype == "bf16" and (cfg.M // cfg.n_heads) in (64, 128)

        def kgroup(site):
            """call site of the library's profile -> the CUDA kernel group it launches"""
            if site.startswith("gemm"):
                return "gemm"
            return "colsum" if site.startswith("colsum") else site

        def bound_of(g):
            """the dense contractions (tcgen05 GEMM, tcgen05 attention) against
            the tensor roof, the routing / movement kernels against HBM; the fp32 SIMT paths
            (f32 parity mode, d_h 16/32) against the FMA pipes."""
            if g == "gemm" or g.startswith("attn"):
                if cfg.dtype == "bf16" and (g == "gemm" or tc_attn):
                    return "tensor", "TFLOP/s", peaks["bf16_tflops_sustained"], "measured sustained bf16"
                return "alu", "TFLOP/s", 148 * 128 * 2 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12, \
                    "148 SMs x 128 FP32 lanes x 2 x max clock"
            return "hbm", "GB/s", peaks["hbm_gbs"], "measured copy"

        # algorithmic work per step of each kernel group (the call sites' FLOPs / bytes from
        # the library's per-launch accounting; identical in every iteration)
        alg = {}
        for p in compute:
            a_ = alg.setdefault(kgroup(p["name"]), {"launches": 0, "flops": 0.0, "bytes": 0.0, "eager_ms": 0.0})
            a_["launches"] += p["launches"]
            a_["flops"] += p["flops"]
            a_["bytes"] += p["bytes"]
            a_["eager_ms"] += p["ms"]
        # device time per step of each group in the steady state: the CUPTI trace of the
        # CUDA-graph replays (rank 0); busy = union of the group's kernel intervals (kernels
        # of one group on different lanes overlap), sum = Σ launch durations
        tl0 = None
        if tl is not None:
            rr = tl["per_rank"] if "per_rank" in tl else [tl]
            tl0 = rr[0] if rr and rr[0] and "groups" in rr[0] else None
        tgroups = tl0["groups"] if tl0 else {}
        tgroups_pdl = tgroups
        # the PDL-off intervals stand for the kernels' execution only where PDL does not
        # change the schedule (the GEMM-bound configs); where it does (latency-bound c2:
        # every launch gap shows), the PDL trace stays the measurement
        if tl_nopdl is not None and "groups" in tl_nopdl and tl0 and \
                tl_nopdl.get("span_us_per_iter", 0) <= 1.05 * tl0.get("span_us_per_iter", 0):
            tgroups = tl_nopdl["groups"]

        def roof(g):
            bound, unit, peak, psrc = bound_of(g)
            a_ = alg[g]
            work = a_["flops"] / 1e12 if unit == "TFLOP/s" else a_["bytes"] / 1e9
            tg = tgroups.get(g)
            if tg and tg["busy_us_per_iter"] > 0:
                busy_s, sum_s, n = tg["busy_us_per_iter"] * 1e-6, tg["sum_us_per_iter"] * 1e-6, tg["launches_per_iter"]
                src = ("CUPTI trace of the CUDA-graph replays, graph captured with PDL off (intervals = execution)"
                       if tgroups is not tgroups_pdl else "CUPTI trace of the CUDA-graph replays")
            else:  # no trace: the eager per-launch event timing (lanes collapsed)
                busy_s = sum_s = a_["eager_ms"] * 1e-3
                n = a_["launches"]
                src = "eager per-launch CUDA events (lanes collapsed)"
            ach = work / busy_s
            # the per-launch roofline of a mixed group: each call site's launches bounded by
            # max(FLOPs / tensor peak, bytes / HBM peak) — the weight-streaming expert GEMMs and
            # the fp32 wgrads sit on the HBM side of the ridge (§6)
            lb_s = 0.0
            for p_ in compute:
                if kgroup(p_["name"]) == g and p_["launches"] > 0:
                    fl, by = p_["flops"] / p_["launches"], p_["bytes"] / p_["launches"]
                    lb_s += p_["launches"] * max(fl / (peaks["bf16_tflops_sustained"] * 1e12) if unit == "TFLOP/s" else 0.0,
                                                 by / (peaks["hbm_gbs"] * 1e9))
            tp = tgroups_pdl.get(g) if tgroups is not tgroups_pdl else None
            extra = {"busy_ms_per_step_pdl_trace": tp["busy_us_per_iter"] * 1e-3} if tp else {}
            extra["per_launch_bound_ms_per_step"] = lb_s * 1e3
            extra["frac_of_per_launch_bound"] = lb_s / busy_s if busy_s > 0 else None
            return {**extra, "bound": bound, "unit": unit, "achieved": ach, "peak": peak, "frac": ach / peak,
                    "peak_source": psrc, "busy_ms_per_step": busy_s * 1e3, "sum_launch_ms_per_step": sum_s * 1e3,
                    "launches_per_step": n, "per_launch_us": sum_s / max(n, 1) * 1e6,
                    "achieved_per_launch": work / sum_s, "timing": src,
                    "algorithmic_per_step": {"flops": a_["flops"], "bytes": a_["bytes"]}}

        key = (lambda g: tgroups[g]["busy_us_per_iter"]) if tgroups else (lambda g: alg[g]["eager_ms"])
        top_g = max((g for g in alg if (g in tgroups or not tgroups)), key=key)
        R_ = roof(top_g)
        per_site = []
        for g in sorted(alg, key=lambda g: -(tgroups[g]["busy_us_per_iter"] if g in tgroups else 0.0))[:12]:
            r_ = roof(g)
            per_site.append({"group": g, "bound": r_["bound"], "achieved": r_["achieved"], "unit": r_["unit"],
                             "frac": r_["frac"], "busy_ms_per_step": r_["busy_ms_per_step"],
                             "launches_per_step": r_["launches_per_step"], "per_launch_us": r_["per_launch_us"]})
        eager_sites = [{"site": p["name"], "us_per_launch": p["ms"] / p["launches"] * 1e3, "launches": p["launches"],
                        "eager_share": p["ms"] / total_ms} for p in sorted(compute, key=lambda p: -p["ms"])[:12]]
        traffic = None
        try:
            tr = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
            traffic = tr.get(args.config, {}).get(top_g, {}).get("dram_bytes_per_launch")
        except Exception:
            pass
        line = {
            "metric": METRIC, "value": tokens / (ms * 1e-3), "unit": "tokens/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
            "config": {"workload": CONFIG_NAMES[args.config], "tokens_per_gpu": cfg.T,
                       "seq_len": cfg.seq_len, "M": cfg.M, "n_heads": cfg.n_heads, "E": cfg.E,
                       "top_k": cfg.top_k, "d_ffn": cfg.d_ffn, "R": cfg.R, "layers": L,
                       "capacity_factor": cfg.capacity_factor, "S_p_bytes": S_p,
                       "parallelism": f"ep{world}+dp{world}", "cuda_graph": not args.no_graph,
                       "compute_streams": args.compute_streams, "schedule": args.schedule,
                       "a2a": args.a2a, "api": "per_block" if args.per_block else "stack",
                       "optimizer": args.optimizer or "excluded (P:304-305)",
                       "l2": "flushed between steps (256 MiB memset outside the event-timed region)"},
            "roofline": {"kernel": top_g, "bound": R_["bound"], "achieved": R_["achieved"], "peak": R_["peak"],
                         "unit": R_["unit"], "frac": R_["frac"], "traffic": traffic,
                         "peak_source": R_["peak_source"], "timing": R_["timing"],
                         "busy_ms_per_step": R_["busy_ms_per_step"],
                         "busy_ms_per_step_pdl_trace": R_.get("busy_ms_per_step_pdl_trace"),
                         "per_launch_bound_ms_per_step": R_.get("per_launch_bound_ms_per_step"),
                         "frac_of_per_launch_bound": R_.get("frac_of_per_launch_bound"),
                         "sum_launch_ms_per_step": R_["sum_launch_ms_per_step"],
                         "launches_per_step": R_["launches_per_step"], "per_launch_us": R_["per_launch_us"],
                         "achieved_per_launch": R_["achieved_per_launch"],
                         "algorithmic_per_step": R_["algorithmic_per_step"],
                         "cross_check": {"busy_ms_per_step": R_["busy_ms_per_step"], "ms_per_step": ms,
                                         "busy_le_step": R_["busy_ms_per_step"] <= ms * 1.05,
                                         "note": "busy = union of the group's kernel intervals per replay "
                                                 "(traced replays run without the L2 flush)"},
                         "groups": per_site, "eager_call_sites": eager_sites},
            "e2e": {"value": tokens / (e2e_ms * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": x0.numel() * x0.element_size() * 2,
                    "d2h_bytes_per_step": dxs[0].numel() * dxs[0].element_size()},
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "exposed_comm": None,
        }
        if tl is not None:
            ranks = tl["per_rank"] if "per_rank" in tl else [tl]

            def valid(r):
                """a usable trace holds about one iteration's kernels per replay and spans
                about one step per replay (CUPTI occasionally drops a rank's records)"""
                return (r and "error" not in r and r["kernels_per_iter"] >= 0.5 * launches_per_step
                        and 0.5 * ms <= r["span_us_per_iter"] / 1e3 <= 4.0 * ms)
            ok = [r for r in ranks if valid(r)]
            if ok and world > 1:
                worst = max(ok, key=lambda r: r["exposed_comm_us_per_iter"])
                med = sorted(ok, key=lambda r: r["exposed_comm_us_per_iter"])[len(ok) // 2]
                line["exposed_comm"] = {
                    "frac_of_comm": worst["exposed_comm_frac_of_comm"],
                    "frac_of_iteration": worst["exposed_comm_frac_of_iter"],
                    "exposed_ms": worst["exposed_comm_us_per_iter"] / 1e3,
                    "comm_busy_ms": worst["comm_busy_us_per_iter"] / 1e3,
                    "median_rank_frac_of_comm": med["exposed_comm_frac_of_comm"],
                    "median_rank_exposed_ms": med["exposed_comm_us_per_iter"] / 1e3,
                    "ranks_valid": len(ok), "ranks": len(ranks),
                    "method": f"CUPTI trace of {args.trace_iters} graph replays (edge iterations "
                              "trimmed); worst valid rank; |union(comm kernels: NCCL, peer-memory A2A) "
                              "minus union(compute kernels)|",
                    # the peer-memory exchange kernel copies, then waits for its peers: counted
                    # only over its transfer time (bytes / 770 GB/s measured peer copy), the
                    # rest is waiting on a slower peer (load imbalance), not communication
                    "transfer_only": {
                        "frac_of_transfer": worst.get("exposed_transfer_frac_of_transfer"),
                        "exposed_ms": worst.get("exposed_transfer_us_per_iter", 0.0) / 1e3,
                        "transfer_ms": worst.get("transfer_comm_us_per_iter", 0.0) / 1e3,
                        "frac_of_iteration": worst.get("exposed_transfer_us_per_iter", 0.0) / 1e3 / ms,
                        "a2a_bytes_per_exchange": a2a_bytes}}
            if ok:
                r0 = ok[0]
                line["timeline"] = {"span_ms": r0["span_us_per_iter"] / 1e3,
                                    "compute_busy_ms": r0["compute_busy_us_per_iter"] / 1e3,
                                    "idle_ms": r0["idle_us_per_iter"] / 1e3,
                                    "kernels_per_iter": r0["kernels_per_iter"]}
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_oracle_baseline(cfg, L)
        if args.profile_json:
            json.dump({"config": args.config, "ms_per_step_eager_profiled": sum(p["ms"] for p in compute),
                       "kernels": sorted(prof, key=lambda p: -p["ms"]), "timeline": tl},
                      open(args.profile_json, "w"), indent=1)
        print(json.dumps(line), flush=True)
    # a CUDA graph that captured NCCL calls must be destroyed before the communicators
    if not args.no_graph:
        del graph, run
    torch.cuda.synchronize()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
