"""Uninitialized-read finder (dev tool): fill most of the free device memory with NaN, free
it back to the driver, then run a stack case through the C ABI (per-block and stack API +
CUDA graph) and report which outputs contain NaN / differ — a read of memory that was never
written in this run then shows up as NaN instead of the zeros of a fresh allocation.
  python tools/probe/poison_run.py [case]   (case: tok | bf16 | f32)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from synth import BlockConfig, gen_replicated, gen_worker  # noqa: E402
from tests.gpu_util import run_stack_gpu  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "tok"
cfg = {"tok": BlockConfig(T=512, seq_len=512, M=256, n_heads=2, E=4, top_k=2, d_ffn=256, R=8, capacity_factor=1.0,
                          causal=1, residual=1, P=1, dtype="bf16"),
       "bf16": BlockConfig(T=1024, seq_len=256, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=4, capacity_factor=1.0,
                           causal=1, residual=1, P=1, dtype="bf16")}[case]


def poison():
    free, _ = torch.cuda.mem_get_info()
    n = int(free * 0.8) // 4
    t = torch.empty(n, dtype=torch.float32, device="cuda")
    t.fill_(float("nan"))
    torch.cuda.synchronize()
    del t
    torch.cuda.empty_cache()


L = 3
reps = [gen_replicated(cfg, block=l) for l in range(L)]
wk = gen_worker(cfg, 0)
wk["forced"] = None
res = {}
for api, graph in (("per_block", False), ("stack", False), ("stack", True)):
    poison()
    g = run_stack_gpu(cfg, reps, wk, compute_streams=cfg.R, api=api, graph=graph)
    res[(api, graph)] = g
    nans = {n: bool(np.isnan(g[n]).any()) for n in ("y", "dx")}
    nans.update({f"{n}{l}": bool(np.isnan(g[n][l]).any()) for n in ("grad_flat", "dw1") for l in range(L)})
    nans.update({f"dxs{l}": bool(np.isnan(g["dxs"][l]).any()) for l in range(L)})
    print(api, "graph" if graph else "eager", "NaN in:", [k for k, v in nans.items() if v] or "none")
ref = res[("per_block", False)]
for key, g in res.items():
    diff = [n for n in ("y", "dx") if not np.array_equal(g[n], ref[n])]
    diff += [f"{n}{l}" for n in ("grad_flat", "dw1") for l in range(L) if not np.array_equal(g[n][l], ref[n][l])]
    diff += [f"dxs{l}" for l in range(L) if not np.array_equal(g["dxs"][l], ref["dxs"][l])]
    print(key, "differs from per_block in:", diff or "nothing")
