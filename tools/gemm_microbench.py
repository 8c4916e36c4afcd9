"""Per-launch device time of the tcgen05 GEMM at the block's shapes, measured inside a
CUDA graph of `reps` back-to-back launches (so host launch cost is excluded), with forced
tile widths and CTA grouping (1 = one CTA per 128-row tile, 2 = CTA pairs with
cta_group::2 UMMAs).  The knobs are per ctx (flowmoe_test.h flowmoe_debug_set).
Prints one JSON line per case.   python tools/gemm_microbench.py [prefix ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2510_00207_b200 as fm  # noqa: E402

SHAPES = {  # name: (M rows, N, K, batch, a_mmajor, b_kmajor, epi)
    "c2_qkv": (256, 768, 256, 1, 0, 0, 0),
    "c2_oproj": (256, 256, 256, 1, 0, 0, 0),
    "c2_e1": (64, 512, 256, 8, 0, 0, 0),
    "c2_e2": (64, 256, 512, 8, 0, 0, 0),
    "c2_dwqkv": (256, 768, 1024, 1, 1, 0, 4),
    "c3_e1": (128, 2048, 1024, 16, 0, 0, 0),
    "c3_qkv": (1024, 3072, 1024, 1, 0, 0, 0),
    "c3_e2": (128, 1024, 2048, 16, 0, 0, 0),
    "c3_dxe": (128, 1024, 2048, 16, 0, 1, 0),
    "c3_oproj": (1024, 1024, 1024, 1, 0, 0, 0),
    "c3_dx": (1024, 1024, 3072, 1, 0, 1, 0),
    "c4_e1": (128, 16384, 4096, 16, 0, 0, 0),
    "c4_qkv": (1024, 12288, 4096, 1, 0, 0, 0),
    "c4_dw1": (4096, 16384, 256, 16, 1, 0, 4),
    # configs[4] DeepSeek-V2-S-shaped (the bench workload): T_r = 512, M = 5120, F = 1536,
    # E = 16 experts x P·C = 256 capacity rows per chunk, K = R·P·C = 512 for the expert wgrads
    "dsv2s_qkv": (512, 15360, 5120, 1, 0, 0, 0),
    "dsv2s_oproj": (512, 5120, 5120, 1, 0, 0, 0),
    "dsv2s_e1": (256, 1536, 5120, 16, 0, 0, 0),
    "dsv2s_e2": (256, 5120, 1536, 16, 0, 0, 0),
    "dsv2s_dgelu": (256, 1536, 5120, 16, 0, 1, 0),
    "dsv2s_dxe": (256, 5120, 1536, 16, 0, 1, 0),
    "dsv2s_dctx": (512, 5120, 5120, 1, 0, 1, 0),
    "dsv2s_dx": (512, 5120, 15360, 1, 0, 1, 0),
    "dsv2s_dw1": (5120, 1536, 512, 16, 1, 0, 4),
    "dsv2s_dw2": (1536, 5120, 512, 16, 1, 0, 4),
    "dsv2s_dwqkv": (5120, 15360, 1024, 1, 1, 0, 4),
    "dsv2s_dwo": (5120, 5120, 1024, 1, 1, 0, 4),
    # with the block's real epilogues: E1 bias + GELU saving GELU'(z) (5), dZ = dH ⊙ aux (6)
    "dsv2s_e1gelu": (256, 1536, 5120, 16, 0, 0, 5),
    "dsv2s_dgelu_mul": (256, 1536, 5120, 16, 0, 1, 6),
}

_CTX = None


def knob_ctx():
    """a small P=1 ctx that carries the GEMM knobs (flowmoe_debug_set is per ctx)"""
    global _CTX
    if _CTX is None:
        _CTX = fm.FlowMoE(fm.BlockShape(B=256, seq_len=64, M=64, n_heads=1, E=2, top_k=1, d_ffn=64, R=1), 0)
    return _CTX


def run(name, reps, bn, pdl, cg=0, sk=0, quiet=False):
    Mr, N, K, batch, am, bk, epi = SHAPES[name]
    dev = torch.device("cuda", 0)
    A = torch.randn(batch, (K if am else Mr), (Mr if am else K), device=dev).to(torch.bfloat16)
    B = torch.randn(batch, (N if bk else K), (K if bk else N), device=dev).to(torch.bfloat16) * 0.05
    C = torch.zeros(batch, Mr, N, device=dev, dtype=torch.float32 if epi == 4 else torch.bfloat16)
    bias = torch.randn(batch, N, device=dev).to(torch.bfloat16) if epi == 5 else None
    aux = torch.randn(batch, Mr, N, device=dev).to(torch.bfloat16) if epi in (5, 6) else None
    ctx = knob_ctx()
    ctx.debug_set(5, bn)
    ctx.debug_set(4, pdl)
    ctx.debug_set(7, cg)
    ctx.debug_set(8, sk)
    kw = dict(M=Mr, N=N, K=K, batch=batch, lda=(Mr if am else K), sA=Mr * K, a_mmajor=am,
              ldb=(K if bk else N), sB=K * N, b_kmajor=bk, ldc=N, sC=Mr * N, epi=epi, bias=bias, aux=aux)
    s = torch.cuda.current_stream()
    fm.test_gemm("bf16", A, B, C, stream=s, ctx=ctx, **kw)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(s)
    with torch.cuda.graph(g, stream=cap, capture_error_mode="thread_local"):
        for _ in range(reps):
            fm.test_gemm("bf16", A, B, C, stream=torch.cuda.current_stream(), ctx=ctx, **kw)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
    flops = 2.0 * Mr * N * K * batch
    if not quiet:
        print(json.dumps({"shape": name, "bn": bn, "cg": cg, "sk": sk, "pdl": pdl, "us_per_launch": round(us, 3),
                          "tflops": round(flops / us / 1e6, 1)}), flush=True)
    del g


def run_plain(name, bn, cg, sk, times=2):
    """`times` plain launches of one forced variant (no graph): what ncu captures"""
    Mr, N, K, batch, am, bk, epi = SHAPES[name]
    dev = torch.device("cuda", 0)
    A = torch.randn(batch, (K if am else Mr), (Mr if am else K), device=dev).to(torch.bfloat16)
    B = torch.randn(batch, (N if bk else K), (K if bk else N), device=dev).to(torch.bfloat16) * 0.05
    C = torch.zeros(batch, Mr, N, device=dev, dtype=torch.float32 if epi == 4 else torch.bfloat16)
    bias = torch.randn(batch, N, device=dev).to(torch.bfloat16) if epi == 5 else None
    aux = torch.randn(batch, Mr, N, device=dev).to(torch.bfloat16) if epi in (5, 6) else None
    ctx = knob_ctx()
    ctx.debug_set(5, bn)
    ctx.debug_set(7, cg)
    ctx.debug_set(8, sk)
    kw = dict(M=Mr, N=N, K=K, batch=batch, lda=(Mr if am else K), sA=Mr * K, a_mmajor=am,
              ldb=(K if bk else N), sB=K * N, b_kmajor=bk, ldc=N, sC=Mr * N, epi=epi, bias=bias, aux=aux)
    for _ in range(times):
        fm.test_gemm("bf16", A, B, C, stream=torch.cuda.current_stream(), ctx=ctx, **kw)
    torch.cuda.synchronize()
    print(json.dumps({"shape": name, "bn": bn, "cg": cg, "sk": sk, "plain_launches": times}), flush=True)


def run_cublas(name, reps):
    """the same contraction through torch (cuBLAS / cuBLASLt, bf16 in, fp32 accumulate; plain
    store, no fused epilogue) in the same graph-of-launches harness: the library baseline"""
    Mr, N, K, batch, am, bk, epi = SHAPES[name]
    dev = torch.device("cuda", 0)
    A = torch.randn(batch, (K if am else Mr), (Mr if am else K), device=dev).to(torch.bfloat16)
    B = torch.randn(batch, (N if bk else K), (K if bk else N), device=dev).to(torch.bfloat16) * 0.05
    At = A.transpose(1, 2) if am else A
    Bt = B.transpose(1, 2) if bk else B
    C = torch.empty(batch, Mr, N, device=dev, dtype=torch.bfloat16)  # bf16 out even for the fp32 wgrads

    def one():
        torch.bmm(At, Bt, out=C)
    s = torch.cuda.current_stream()
    one()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    cap.wait_stream(s)
    with torch.cuda.graph(g, stream=cap):
        for _ in range(reps):
            one()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / (5 * reps)
    print(json.dumps({"shape": name, "impl": "cublas (torch.bmm)", "us_per_launch": round(us, 3),
                      "tflops": round(2.0 * Mr * N * K * batch / us / 1e6, 1)}), flush=True)
    del g


if __name__ == "__main__":
    pref = tuple(sys.argv[1:]) or ("",)
    for name in SHAPES:
        if not name.startswith(pref):
            continue
        reps = 200 if name.startswith("c2") else (50 if name.startswith("c3") else 10)
        if os.environ.get("ONLY"):  # variants "cg,bn,sk;cg,bn,sk" launched twice each, no graph (ncu runs)
            for spec in os.environ["ONLY"].split(";"):
                cg, bn, sk = (int(v) for v in spec.split(","))
                run_plain(name, bn, cg, sk)
            continue
        run(name, reps, 0, 1, 0, quiet=True)  # warm-up (clocks, allocator, module load)
        run(name, reps, 0, 1, 0)  # the library's automatic choice
        for cg, bn, sk in ((1, 128, 0), (1, 192, 0), (1, 256, 0), (2, 128, 0), (2, 256, 0), (2, 512, 0),
                           (1, 256, 2), (2, 256, 2)):
            run(name, reps, bn, 1, cg, sk)
        if os.environ.get("CUBLAS", "1") == "1":
            run_cublas(name, reps)
