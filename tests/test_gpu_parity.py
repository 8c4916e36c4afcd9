"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on the
same seeded synth inputs.  Tolerances (BASELINE.json north_star): routing
indices / counts / positions bit-exact given identical logits; fp32 values
rel <= 1e-4; bf16 with fp32 accumulation rel <= 2e-2, rel = max|g-r|/max|r|."""
import ctypes

import numpy as np
import pytest

import oracle as o
import paper_2510_00207_b200 as fm
from synth import PRESETS, BlockConfig, gen_replicated, gen_worker
from tests.gpu_util import expert_grads, oracle_block, rel, run_block_gpu

pytestmark = pytest.mark.gpu

TOL = {"f32": 1e-4, "bf16": 2e-2}

CASES = {
    # configs[0] at P=1 (all 4 experts local), capacity drops (f=1.0)
    "c1_f32": PRESETS["c1"].replace(P=1),
    "c1_f32_dropless_causal_resid": PRESETS["c1_dropless"].replace(P=1, causal=1, residual=1),
    "f32_k1": BlockConfig(T=256, seq_len=64, M=64, n_heads=2, E=8, top_k=1, d_ffn=96, R=4,
                          capacity_factor=1.0, causal=1, residual=0, P=1, dtype="f32"),
    # bf16, several tiles + ragged tails in every GEMM dimension
    "bf16_small": BlockConfig(T=512, seq_len=128, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=2,
                              capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    "bf16_ragged": BlockConfig(T=384, seq_len=96, M=192, n_heads=3, E=4, top_k=2, d_ffn=328, R=2,
                               capacity_factor=1.25, causal=0, residual=0, P=1, dtype="bf16"),
    "bf16_k3_dh128": BlockConfig(T=256, seq_len=128, M=256, n_heads=2, E=16, top_k=3, d_ffn=256,
                                 R=2, capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    # configs[1]: the bench workload (GPT2-Tiny-MoE-shaped, R=4), full size
    "c2_bench": PRESETS["c2"],
    # long sequences: several 128-row attention tiles, causal diagonal tiles, d_h 128 / 64
    "bf16_long_causal_dh128": BlockConfig(T=1024, seq_len=512, M=256, n_heads=2, E=4, top_k=2,
                                          d_ffn=256, R=2, capacity_factor=1.0, causal=1, residual=1,
                                          P=1, dtype="bf16"),
    "bf16_long_dh64_ragged": BlockConfig(T=768, seq_len=384, M=256, n_heads=4, E=4, top_k=2,
                                         d_ffn=256, R=2, capacity_factor=1.0, causal=0, residual=0,
                                         P=1, dtype="bf16"),
    "bf16_ragged_seq_causal": BlockConfig(T=400, seq_len=200, M=128, n_heads=2, E=4, top_k=2,
                                          d_ffn=256, R=2, capacity_factor=1.0, causal=1, residual=1,
                                          P=1, dtype="bf16"),
    # gate kernel variants: wide E with k up to 8 and an 8-CTA cluster split over M
    # (peer slices pushed with st.async), E = 64, E = 2 with k = 1, and a chunk whose
    # routing scan exceeds the per-thread register segment (T_r·k = 4096 slots)
    "gate_e32_k8": BlockConfig(T=512, seq_len=128, M=512, n_heads=4, E=32, top_k=8, d_ffn=128, R=2,
                               capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    "gate_e64_k4": BlockConfig(T=512, seq_len=128, M=256, n_heads=4, E=64, top_k=4, d_ffn=64, R=2,
                               capacity_factor=1.5, causal=0, residual=1, P=1, dtype="bf16"),
    "gate_e2_k1": BlockConfig(T=256, seq_len=64, M=256, n_heads=4, E=2, top_k=1, d_ffn=128, R=2,
                              capacity_factor=1.0, causal=1, residual=0, P=1, dtype="bf16"),
    "scan_wide_chunk": BlockConfig(T=4096, seq_len=256, M=128, n_heads=2, E=8, top_k=2, d_ffn=128, R=2,
                                   capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    # T_r·k = 9216 slots > 32 per thread of the fused scan: its streaming (non-register) path
    "scan_beyond_reg": BlockConfig(T=4608, seq_len=256, M=128, n_heads=2, E=8, top_k=4, d_ffn=128, R=2,
                                   capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    # k = 8 of 16 with wide rows (the dsv2s routing shape at a small M): wide gather kernels
    "bf16_k8_wide": BlockConfig(T=512, seq_len=256, M=512, n_heads=4, E=16, top_k=8, d_ffn=256, R=2,
                                capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
}


def _check_block(cfg, forced=True, compute_streams=1):
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    g = run_block_gpu(cfg, rep, wk, forced=forced, compute_streams=compute_streams)
    ys, dxs, gflat, eg, st = oracle_block(cfg, rep, [wk], forced=forced)
    tol = TOL[cfg.dtype]
    res = {"y": rel(g["y"], ys[0]), "dx": rel(g["dx"], dxs[0]),
           "grad_flat": rel(g["grad_flat"], gflat)}
    ref_e = expert_grads(eg, 0, cfg.E)
    for n in ("dw1", "db1", "dw2", "db2"):
        res[n] = rel(g[n], ref_e[n])
    M = cfg.M
    res["dWqkv"] = rel(g["grad_flat"][:3 * M * M], gflat[:3 * M * M])
    res["dWo"] = rel(g["grad_flat"][3 * M * M:4 * M * M], gflat[3 * M * M:4 * M * M])
    res["dWg"] = rel(g["grad_flat"][4 * M * M:], gflat[4 * M * M:])
    bad = {k: v for k, v in res.items() if not v <= tol}
    assert not bad, f"rel errors above {tol}: {bad} (all: {res})"
    # routing under forced indices: identical indices and positions
    ro = st.route[0]
    assert np.array_equal(g["idx"], ro.idx)
    assert np.array_equal(g["pos"], np.where(ro.kept, ro.pos, -1))
    assert np.array_equal(g["counts"], ro.counts)
    res["_gpu"] = g
    return res


@pytest.mark.parametrize("name", list(CASES))
def test_block_parity_forced_routing(name):
    _check_block(CASES[name])


@pytest.mark.parametrize("name", ["bf16_small", "bf16_k8_wide", "bf16_ragged"])
def test_block_parity_cta_pair_gemms(name, monkeypatch):
    """Every GEMM of the block (forward, dgrads, fp32 wgrads) on CTA pairs (cta_group::2,
    forced through the per-ctx knob) vs the oracle; and bit-identical to itself with R lanes."""
    monkeypatch.setenv("FLOWMOE_FORCE_CG2", "1")
    _check_block(CASES[name])


# Token chunks (reading Q1'): R exceeds the number of sequences, every chunk is a causal
# slice of one sequence (chunked prefill).  Chunk offsets on and off the 128-row tiles.
TOK_CASES = {
    "tok_bf16_dh64": BlockConfig(T=512, seq_len=256, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=4,
                                 capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    "tok_bf16_dh128_r8": BlockConfig(T=512, seq_len=512, M=256, n_heads=2, E=4, top_k=2, d_ffn=256, R=8,
                                     capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    "tok_bf16_ragged": BlockConfig(T=384, seq_len=192, M=128, n_heads=2, E=4, top_k=2, d_ffn=256, R=4,
                                   capacity_factor=1.25, causal=1, residual=0, P=1, dtype="bf16"),
    "tok_f32_dh16": BlockConfig(T=256, seq_len=128, M=64, n_heads=4, E=4, top_k=2, d_ffn=128, R=8,
                                capacity_factor=1.0, causal=1, residual=1, P=1, dtype="f32"),
    "tok_f32_dh32": BlockConfig(T=192, seq_len=96, M=64, n_heads=2, E=4, top_k=2, d_ffn=96, R=6,
                                capacity_factor=0.0, causal=1, residual=0, P=1, dtype="f32"),
}


@pytest.mark.parametrize("name", list(TOK_CASES))
def test_token_chunk_parity(name):
    """One lane (the paper's serial order) and R lanes (cross-lane QKV / dctx events)
    both match the oracle, and each other bit for bit."""
    cfg = TOK_CASES[name]
    one = _check_block(cfg, compute_streams=1)["_gpu"]
    many = _check_block(cfg, compute_streams=cfg.R)["_gpu"]
    for n in ("y", "dx", "grad_flat", "dw1", "db1", "dw2", "db2"):
        assert np.array_equal(one[n], many[n]), n


@pytest.mark.parametrize("name", ["c1_f32", "bf16_small", "c2_bench", "bf16_k3_dh128", "f32_k1",
                                  "gate_e32_k8", "gate_e64_k4", "gate_e2_k1", "scan_wide_chunk",
                                  "scan_beyond_reg", "bf16_k8_wide"])
def test_routing_bitexact_given_gpu_logits(name):
    """Natural routing: the oracle routes from the GPU's own fp32 logits; indices,
    positions and per-chunk counts must match bit for bit, weights to fp32 rounding."""
    cfg = CASES[name]
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    g = run_block_gpu(cfg, rep, wk, forced=False)
    ro = o.route_worker(cfg, None, None, logits=g["logits"].astype(np.float64))
    assert np.array_equal(g["idx"], ro.idx)
    assert np.array_equal(g["pos"], np.where(ro.kept, ro.pos, -1))
    assert np.array_equal(g["counts"], ro.counts)
    assert np.max(np.abs(g["w"] - ro.w)) < 1e-6
    # and the logits themselves match the oracle's A·Wg to the dtype tolerance
    ys, dxs, gflat, eg, st = oracle_block(cfg, rep, [wk], forced=False)
    assert rel(g["logits"], st.route[0].logits) <= TOL[cfg.dtype]


@pytest.mark.parametrize("name", ["bf16_small", "gate_e32_k8", "c1_f32", "gate_e64_k4"])
def test_routing_crafted_ties(name):
    """Reading Q4 on the GPU with ties forced: duplicated gate columns give bit-equal
    logits, so top-k must pick the lower expert index; and an all-equal gate (every
    column the same) must route every token to experts 0..k-1 with weights 1/k."""
    cfg = CASES[name]
    wk = gen_worker(cfg, 0)
    rep = gen_replicated(cfg)
    E = cfg.E
    wg = rep["wg"].copy()
    pairs = [(0, E - 1), (1, E // 2 + 1), (2, 3)] if E >= 8 else [(0, E - 1)]
    for lo, hi in pairs:
        wg[:, hi] = wg[:, lo]
    g = run_block_gpu(cfg, dict(rep, wg=wg), wk, forced=False)
    for lo, hi in pairs:
        assert np.array_equal(g["logits"][:, lo], g["logits"][:, hi]), "duplicated columns must tie exactly"
    ro = o.route_worker(cfg, None, None, logits=g["logits"].astype(np.float64))
    assert np.array_equal(g["idx"], ro.idx)
    assert np.array_equal(g["pos"], np.where(ro.kept, ro.pos, -1))
    assert np.array_equal(g["counts"], ro.counts)
    decided = sum(int(np.sum(np.any(g["idx"] == lo, axis=1) & ~np.any(g["idx"] == hi, axis=1)))
                  for lo, hi in pairs)
    assert decided > 0, "some token must sit on a tie at the k-th place"
    for lo, hi in pairs:  # the higher index never wins a tie against the lower one ...
        assert not np.any(np.any(g["idx"] == hi, axis=1) & ~np.any(g["idx"] == lo, axis=1))
        both = np.any(g["idx"] == lo, axis=1) & np.any(g["idx"] == hi, axis=1)
        slot = lambda e: np.argmax(g["idx"][both] == e, axis=1)  # noqa: E731
        assert np.all(slot(lo) < slot(hi))  # ... and takes the earlier slot when both are picked
    g = run_block_gpu(cfg, dict(rep, wg=np.repeat(rep["wg"][:, :1], E, axis=1)), wk, forced=False)
    assert np.array_equal(g["idx"], np.tile(np.arange(cfg.top_k, dtype=np.int32), (cfg.T, 1)))
    want_w = 1.0 / cfg.top_k if cfg.top_k > 1 else 1.0 / E
    assert np.max(np.abs(g["w"] - want_w)) < 1e-6
    ro = o.route_worker(cfg, None, None, logits=g["logits"].astype(np.float64))
    assert np.array_equal(g["pos"], np.where(ro.kept, ro.pos, -1))
    assert np.array_equal(g["counts"], ro.counts)


def test_skewed_routing_with_drops_bf16():
    """Zipf-skewed expert popularity (input recipe 'skew'): uneven loads and drops."""
    cfg = CASES["bf16_small"]
    rep = gen_replicated(cfg, skew=True)
    wk = gen_worker(cfg, 0, skew=True)
    g = run_block_gpu(cfg, rep, wk, forced=False)
    ro = o.route_worker(cfg, None, None, logits=g["logits"].astype(np.float64))
    assert (~ro.kept).sum() > 0.1 * ro.kept.size, "skew must force capacity drops"
    assert np.array_equal(g["pos"], np.where(ro.kept, ro.pos, -1))
    assert np.array_equal(g["counts"], ro.counts)
    wk2 = dict(wk, forced_idx=ro.idx)
    g2 = run_block_gpu(cfg, rep, wk2, forced=True)
    ys, dxs, gflat, eg, st = oracle_block(cfg, rep, [wk2], forced=True)
    assert rel(g2["y"], ys[0]) <= TOL["bf16"]
    assert rel(g2["dx"], dxs[0]) <= TOL["bf16"]
    assert rel(g2["grad_flat"], gflat) <= TOL["bf16"]


def test_chunked_equals_unchunked_on_gpu():
    """Pipelining (R chunks) does not change the result: GPU R=4 vs R=1, dropless."""
    base = BlockConfig(T=256, seq_len=32, M=64, n_heads=4, E=4, top_k=2, d_ffn=128, R=1,
                       capacity_factor=0.0, causal=1, residual=1, P=1, dtype="f32")
    rep = gen_replicated(base)
    wk = gen_worker(base, 0)
    a = run_block_gpu(base, rep, wk)
    b = run_block_gpu(base.replace(R=4), rep, wk)
    for n in ("y", "dx"):
        assert np.array_equal(a[n], b[n]), n
    for n in ("grad_flat", "dw1", "db1", "dw2", "db2"):
        assert rel(b[n], a[n]) <= 1e-5, n


def test_empty_expert_and_all_tokens_one_expert():
    """Degenerate routing: every token forced to experts {0,1}; experts 2..7 get
    no rows (their grads stay exactly 0), most slots of 0/1 are dropped."""
    cfg = CASES["bf16_small"].replace(capacity_factor=1.0)
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    wk["forced_idx"] = np.tile(np.array([[0, 1]], dtype=np.int32), (cfg.T, 1))
    g = run_block_gpu(cfg, rep, wk)
    ys, dxs, gflat, eg, st = oracle_block(cfg, rep, [wk])
    assert rel(g["y"], ys[0]) <= TOL["bf16"]
    assert rel(g["dx"], dxs[0]) <= TOL["bf16"]
    assert np.all(g["dw1"][2:] == 0) and np.all(g["db2"][2:] == 0)


GEMM_SHAPES = [(200, 320, 136, 2), (128, 96, 64, 1), (296, 200, 520, 3), (64, 512, 256, 8)]  # rows, N, K multiple of 8 (TMA 16-B strides)


_KNOB_CTX = {}


def knob_ctx(cg=0, bn=0, sk=0):
    """a small ctx carrying GEMM knobs (flowmoe_test.h: per-ctx debug keys 5, 7 and 8)"""
    import paper_2510_00207_b200 as fm
    if (cg, bn, sk) not in _KNOB_CTX:
        c = fm.FlowMoE(fm.BlockShape(B=256, seq_len=64, M=64, n_heads=1, E=2, top_k=1, d_ffn=64, R=1), 0)
        c.debug_set(7, cg)
        c.debug_set(5, bn)
        c.debug_set(8, sk)
        _KNOB_CTX[(cg, bn, sk)] = c
    return _KNOB_CTX[(cg, bn, sk)]


GEMM_CG = [(0, 0), (0, 192), (2, 256), (2, 128), (2, 512)]  # automatic; 192-column tiles; CTA pairs (cta_group::2) with 256 / 128 / 512 columns


@pytest.mark.parametrize("cg,bn", GEMM_CG)
@pytest.mark.parametrize("a_mmajor,b_kmajor", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_gemm_tc_layouts_vs_fp64(a_mmajor, b_kmajor, shape, cg, bn):
    """tcgen05 GEMM (bf16 in, fp32 TMEM accum) against the fp64 product of the
    same bf16 inputs; store epilogue (bf16 out) and fp32 accumulate epilogue; single-CTA
    tiles and CTA pairs (ragged M: the pair's second CTA partly or wholly past the rows;
    ragged N: the second CTA's B half past the columns)."""
    import torch
    import paper_2510_00207_b200 as fm
    ctx = knob_ctx(cg, bn)
    Mr, N, K, batch = shape
    rng = np.random.default_rng(sum(shape) + 7 * a_mmajor + 3 * b_kmajor)
    A = rng.standard_normal((batch, Mr, K))
    B = rng.standard_normal((batch, K, N))
    dev = torch.device("cuda", 0)
    a_store = A.transpose(0, 2, 1).copy() if a_mmajor else A
    b_store = B.transpose(0, 2, 1).copy() if b_kmajor else B
    At = fm.to_device(a_store, "bf16", dev)
    Bt = fm.to_device(b_store, "bf16", dev)
    Ar = fm.to_host_f64(At)
    Br = fm.to_host_f64(Bt)
    Ar = Ar.transpose(0, 2, 1) if a_mmajor else Ar
    Br = Br.transpose(0, 2, 1) if b_kmajor else Br
    ref = Ar @ Br
    lda = Mr if a_mmajor else K
    ldb = K if b_kmajor else N
    C = torch.zeros((batch, Mr, N), dtype=torch.bfloat16, device=dev)
    fm.test_gemm("bf16", At, Bt, C, M=Mr, N=N, K=K, batch=batch, lda=lda, sA=Mr * K,
                 a_mmajor=a_mmajor, ldb=ldb, sB=K * N, b_kmajor=b_kmajor, ldc=N, sC=Mr * N, ctx=ctx)
    C32 = torch.ones((batch, Mr, N), dtype=torch.float32, device=dev)
    fm.test_gemm("bf16", At, Bt, C32, M=Mr, N=N, K=K, batch=batch, lda=lda, sA=Mr * K,
                 a_mmajor=a_mmajor, ldb=ldb, sB=K * N, b_kmajor=b_kmajor, ldc=N, sC=Mr * N, epi=3, ctx=ctx)
    torch.cuda.synchronize()
    assert rel(fm.to_host_f64(C), ref) <= 1e-2
    assert rel(C32.cpu().numpy().astype(np.float64) - 1.0, ref) <= 1e-5


# rows, N, K, batch: fewer tiles than units (all stream-K), ragged, batched, and whole waves
# plus a stream-K remainder (768 x 7936: 93 pair tiles = 74 whole + 19 cut)
SK_SHAPES = [(512, 2560, 4096, 1), (520, 1000, 3000, 1), (256, 1536, 2048, 2), (768, 7936, 1024, 1)]


@pytest.mark.parametrize("cg,bn", [(2, 256), (1, 256)])
@pytest.mark.parametrize("b_kmajor", [0, 1])
@pytest.mark.parametrize("shape", SK_SHAPES)
def test_gemm_streamk_vs_fp64(shape, b_kmajor, cg, bn):
    """Stream-K GEMM (every pair / CTA the same share of the flattened (tile, k-block) space;
    tiles cut between units summed by the epilogue's fix-up in segment order): against the
    fp64 product with the residual epilogue, ragged M / N / K, batched; two calls bit-identical
    (ordered fix-up; the per-tile counters reset themselves)."""
    import torch
    import paper_2510_00207_b200 as fm
    ctx = knob_ctx(cg, bn, 2)
    Mr, N, K, batch = shape
    rng = np.random.default_rng(Mr + N + K + b_kmajor + cg)
    dev = torch.device("cuda", 0)
    A = fm.to_device(rng.standard_normal((batch, Mr, K)) / 8, "bf16", dev)
    Bm = rng.standard_normal((batch, K, N))
    Bt = fm.to_device(Bm.transpose(0, 2, 1).copy() if b_kmajor else Bm, "bf16", dev)
    res = fm.to_device(rng.standard_normal((batch, Mr, N)), "bf16", dev)
    Br = fm.to_host_f64(Bt)
    ref = fm.to_host_f64(A) @ (Br.transpose(0, 2, 1) if b_kmajor else Br)
    kw = dict(M=Mr, N=N, K=K, batch=batch, lda=K, sA=Mr * K, ldb=K if b_kmajor else N, sB=K * N,
              b_kmajor=b_kmajor, ldc=N, sC=Mr * N, ctx=ctx)
    C = torch.full((batch, Mr, N), 3.0, dtype=torch.bfloat16, device=dev)
    fm.test_gemm("bf16", A, Bt, C, resid=res, **kw)
    C2 = torch.full_like(C, -1.0)
    fm.test_gemm("bf16", A, Bt, C2, resid=res, **kw)
    C32 = torch.ones((batch, Mr, N), dtype=torch.float32, device=dev)  # fp32 accumulate (wgrads)
    fm.test_gemm("bf16", A, Bt, C32, epi=3, **kw)
    torch.cuda.synchronize()
    assert rel(fm.to_host_f64(C), ref + fm.to_host_f64(res)) <= 1e-2
    assert torch.equal(C, C2)
    assert rel(C32.cpu().numpy().astype(np.float64) - 1.0, ref) <= 1e-5


def test_gemm_streamk_epilogues():
    """The fused epilogues run on the fix-up's sum: bias+GELU (Z saved / GELU' saved),
    dGELU, aux multiply, fp32 store, on a stream-K pair GEMM with tiles cut between units."""
    import torch
    import paper_2510_00207_b200 as fm
    ctx = knob_ctx(2, 256, 2)
    Mr, N, K, batch = 256, 1536, 2048, 2
    rng = np.random.default_rng(5)
    dev = torch.device("cuda", 0)
    A = fm.to_device(rng.standard_normal((batch, Mr, K)) / 16, "bf16", dev)
    B = fm.to_device(rng.standard_normal((batch, K, N)) / 4, "bf16", dev)
    bias = fm.to_device(rng.standard_normal((batch, N)), "bf16", dev)
    ref = fm.to_host_f64(A) @ fm.to_host_f64(B)
    kw = dict(M=Mr, N=N, K=K, batch=batch, lda=K, sA=Mr * K, ldb=N, sB=K * N, ldc=N, sC=Mr * N, ctx=ctx)
    C = torch.empty((batch, Mr, N), dtype=torch.bfloat16, device=dev)
    Z = torch.empty_like(C)
    fm.test_gemm("bf16", A, B, C, epi=1, bias=bias, aux=Z, **kw)
    torch.cuda.synchronize()
    z = ref + fm.to_host_f64(bias)[:, None, :]
    assert rel(fm.to_host_f64(Z), z) <= 1e-2
    assert rel(fm.to_host_f64(C), o.gelu(fm.to_host_f64(Z))) <= 1e-2
    fm.test_gemm("bf16", A, B, C, epi=2, aux=Z, **kw)
    torch.cuda.synchronize()
    assert rel(fm.to_host_f64(C), ref * o.gelu_grad(fm.to_host_f64(Z))) <= 1e-2
    D = torch.empty_like(C)
    fm.test_gemm("bf16", A, B, C, epi=5, bias=bias, aux=D, **kw)
    torch.cuda.synchronize()
    zb = fm.to_host_f64(Z)
    assert rel(fm.to_host_f64(C), o.gelu(zb)) <= 1e-2
    assert rel(fm.to_host_f64(D), o.gelu_grad(zb)) <= 1e-2
    fm.test_gemm("bf16", A, B, C, epi=6, aux=D, **kw)
    F = torch.full((batch, Mr, N), 9.0, dtype=torch.float32, device=dev)
    fm.test_gemm("bf16", A, B, F, epi=4, **kw)
    torch.cuda.synchronize()
    assert rel(fm.to_host_f64(C), ref * fm.to_host_f64(D)) <= 1e-2
    assert rel(F.cpu().numpy().astype(np.float64), ref) <= 1e-5


@pytest.mark.parametrize("cg", [0, 1, 2])
@pytest.mark.parametrize("epi", [3, 4])
def test_gemm_tc_wgrad_variant_vs_fp64(epi, cg):
    """The write-bound wgrad shape (fp32 out, K <= 256, >= 4·148 tiles of 256 columns) on an
    m-major A like the expert dW, ragged N and K, against the fp64 product: store (4) and
    accumulate (3); automatic (CTA pairs), single CTAs (cg = 1: the 3-stage ring with
    double-buffered epilogue staging) and forced pairs."""
    import torch
    import paper_2510_00207_b200 as fm
    Mr, N, K = 2048, 9480, 200  # 16 x 38 = 608 tiles
    rng = np.random.default_rng(11 + epi)
    dev = torch.device("cuda", 0)
    At = fm.to_device(rng.standard_normal((1, K, Mr)), "bf16", dev)  # A stored m-major [K][M]
    Bt = fm.to_device(rng.standard_normal((1, K, N)), "bf16", dev)
    ref = fm.to_host_f64(At)[0].T @ fm.to_host_f64(Bt)[0]
    C = torch.full((1, Mr, N), 0.5 if epi == 3 else 7.0, dtype=torch.float32, device=dev)
    fm.test_gemm("bf16", At, Bt, C, M=Mr, N=N, K=K, batch=1, lda=Mr, sA=Mr * K, a_mmajor=1,
                 ldb=N, sB=K * N, ldc=N, sC=Mr * N, epi=epi, ctx=knob_ctx(cg))
    torch.cuda.synchronize()
    got = C[0].cpu().numpy().astype(np.float64) - (0.5 if epi == 3 else 0.0)
    assert rel(got, ref) <= 1e-5


@pytest.mark.parametrize("cg,bn", GEMM_CG)
def test_gemm_tc_epilogues(cg, bn):
    import torch
    import paper_2510_00207_b200 as fm
    ctx = knob_ctx(cg, bn)
    Mr, N, K, batch = 448, 384, 128, 2
    rng = np.random.default_rng(3)
    dev = torch.device("cuda", 0)
    A = fm.to_device(rng.standard_normal((batch, Mr, K)) / 8, "bf16", dev)
    B = fm.to_device(rng.standard_normal((batch, K, N)), "bf16", dev)
    bias = fm.to_device(rng.standard_normal((batch, N)), "bf16", dev)
    res = fm.to_device(rng.standard_normal((batch, Mr, N)), "bf16", dev)
    ref = fm.to_host_f64(A) @ fm.to_host_f64(B)
    kw = dict(M=Mr, N=N, K=K, batch=batch, lda=K, sA=Mr * K, ldb=N, sB=K * N, ldc=N, sC=Mr * N)
    C = torch.empty((batch, Mr, N), dtype=torch.bfloat16, device=dev)
    fm.test_gemm("bf16", A, B, C, epi=0, bias=bias, resid=res, **kw, ctx=ctx)
    want = ref + fm.to_host_f64(bias)[:, None, :] + fm.to_host_f64(res)
    assert rel(fm.to_host_f64(C), want) <= 1e-2
    Z = torch.empty_like(C)
    fm.test_gemm("bf16", A, B, C, epi=1, bias=bias, aux=Z, **kw, ctx=ctx)
    z = ref + fm.to_host_f64(bias)[:, None, :]
    assert rel(fm.to_host_f64(Z), z) <= 1e-2
    assert rel(fm.to_host_f64(C), o.gelu(fm.to_host_f64(Z))) <= 1e-2
    fm.test_gemm("bf16", A, B, C, epi=2, aux=Z, **kw, ctx=ctx)
    torch.cuda.synchronize()
    assert rel(fm.to_host_f64(C), ref * o.gelu_grad(fm.to_host_f64(Z))) <= 1e-2
    # the expert FFN pair: forward saves GELU'(z), backward multiplies by it
    D = torch.empty_like(C)
    fm.test_gemm("bf16", A, B, C, epi=5, bias=bias, aux=D, **kw, ctx=ctx)
    torch.cuda.synchronize()
    zb = fm.to_host_f64(Z)  # bf16(acc + bias) from the epi=1 call, same inputs
    assert rel(fm.to_host_f64(C), o.gelu(zb)) <= 1e-2
    assert rel(fm.to_host_f64(D), o.gelu_grad(zb)) <= 1e-2
    fm.test_gemm("bf16", A, B, C, epi=6, aux=D, **kw, ctx=ctx)
    torch.cuda.synchronize()
    assert rel(fm.to_host_f64(C), ref * fm.to_host_f64(D)) <= 1e-2


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_grad_modes_overwrite_and_accumulate(dtype):
    """OVERWRITE ignores (garbage) buffer contents; ACCUMULATE adds: two backward
    calls give twice the grads (P=1, so the AR is the identity)."""
    cfg = (CASES["c1_f32"] if dtype == "f32" else CASES["bf16_small"])
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    ys, dxs, gflat, eg, st = oracle_block(cfg, rep, [wk])
    ref_e = expert_grads(eg, 0, cfg.E)
    g = run_block_gpu(cfg, rep, wk, grad_mode="overwrite", grad_fill=1e6)
    assert rel(g["grad_flat"], gflat) <= TOL[dtype]
    for n in ("dw1", "db1", "dw2", "db2"):
        assert rel(g[n], ref_e[n]) <= TOL[dtype], n
    g1 = run_block_gpu(cfg, rep, wk, grad_mode="accumulate")
    g2 = run_block_gpu(cfg, rep, wk, grad_mode="accumulate", repeat_bwd=2)
    for n in ("grad_flat", "dw1", "db1", "dw2", "db2"):
        assert rel(g2[n], 2.0 * g1[n]) <= 1e-6, n


@pytest.mark.parametrize("name", ["c2_bench", "c1_f32", "bf16_long_dh64_ragged"])
def test_compute_lanes_bitwise_identical(name):
    """Chunks' compute tasks on min(n, R) streams give bit-identical results to the
    single compute stream (no atomics; every output has one writer)."""
    cfg = CASES[name]
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    a = run_block_gpu(cfg, rep, wk, compute_streams=1)
    b = run_block_gpu(cfg, rep, wk, compute_streams=cfg.R)
    for n in ("y", "dx", "grad_flat", "dw1", "db1", "dw2", "db2", "logits", "idx", "pos", "counts"):
        assert np.array_equal(a[n], b[n]), n


@pytest.mark.parametrize("schedule", ["flowmoe_ar", "flowmoe_at", "pipe_moe"])
@pytest.mark.parametrize("lanes", [1, 4])
def test_schedule_policies_bitwise_identical(schedule, lanes):
    """The Table 6 policies change only the schedule (AT split or not, AR pipelined or
    centralized): same effective R gives bit-identical results (P=1)."""
    cfg = CASES["c2_bench"]
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    a = run_block_gpu(cfg, rep, wk, compute_streams=lanes)
    b = run_block_gpu(cfg, rep, wk, compute_streams=lanes, schedule=schedule)
    for n in ("y", "dx", "grad_flat", "dw1", "db1", "dw2", "db2", "idx", "pos", "counts"):
        assert np.array_equal(a[n], b[n]), n


def test_vanilla_ep_is_the_unchunked_block():
    """VANILLA_EP runs the block as one chunk (R = 1, capacity over all tokens)."""
    cfg = CASES["bf16_small"]
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    g = run_block_gpu(cfg, rep, wk, schedule="vanilla_ep")
    ys, dxs, gflat, eg, st = oracle_block(cfg.replace(R=1), rep, [wk])
    assert rel(g["y"], ys[0]) <= TOL["bf16"]
    assert rel(g["dx"], dxs[0]) <= TOL["bf16"]
    assert rel(g["grad_flat"], gflat) <= TOL["bf16"]
    assert np.array_equal(g["counts"], st.route[0].counts)


def check_chain_per_block(cfg, reps, forced, dy_top, g):
    from tests.gpu_util import chain_per_block_errors
    res = chain_per_block_errors(cfg, reps, forced, dy_top, g)
    bad = {k: v for k, v in res.items() if not v <= TOL[cfg.dtype]}
    assert not bad, (bad, res)
    return res


@pytest.mark.parametrize("dtype,lanes,graph", [("f32", 1, False), ("bf16", 4, False), ("bf16", 4, True),
                                               ("f32", 2, True)])
def test_block_stack_chain_parity(dtype, lanes, graph):
    """3 chained blocks (different weights, forced routing): every block's forward output,
    backward dx and grads vs the oracle run on that block's GPU inputs (per-block
    tolerance); f32 also end to end.  Exercises cross-block reuse of the ctx workspaces,
    compute lanes, the overlapped weight-grad stream, CUDA-graph replay."""
    from tests.gpu_util import run_stack_gpu
    base = CASES["c2_bench"] if dtype == "bf16" else CASES["c1_f32"].replace(R=4, residual=1, causal=1)
    cfg = base
    L = 3
    reps = [gen_replicated(cfg, block=l) for l in range(L)]
    wk = gen_worker(cfg, 0)
    wk["forced"] = [gen_worker(cfg, 0, block=l)["forced_idx"] for l in range(L)]
    g = run_stack_gpu(cfg, reps, wk, compute_streams=lanes, graph=graph)
    check_chain_per_block(cfg, reps, [wk["forced"]], [wk["dy"]], g)
    if dtype == "bf16":  # lanes and graph replay change nothing, bit for bit
        ref = run_stack_gpu(cfg, reps, wk, compute_streams=1, graph=False)
        for n in ("y", "dx"):
            assert np.array_equal(g[n], ref[n]), n
        for l in range(L):
            assert np.array_equal(g["grad_flat"][l], ref["grad_flat"][l]) and np.array_equal(g["dw1"][l], ref["dw1"][l])
        return
    # fp32: the whole chain end to end at the fp32 tolerance as well
    xs, sts = [wk["x"]], []
    for l in range(L):
        ys, st = o.block_forward(cfg, reps[l], [xs[-1]], [wk["forced"][l]])
        xs.append(ys[0])
        sts.append(st)
    dy = wk["dy"]
    for l in reversed(range(L)):
        dxs, gflat, eg = o.block_backward(cfg, reps[l], sts[l], [dy])
        assert rel(g["grad_flat"][l], gflat) <= TOL[dtype], l
        dy = dxs[0]
    assert rel(g["y"], xs[-1]) <= TOL[dtype]
    assert rel(g["dx"], dy) <= TOL[dtype]


@pytest.mark.parametrize("schedule", ["flowmoe_ar", "pipe_moe", "flowmoe_at"])
@pytest.mark.parametrize("graph", [False, True])
def test_stack_api_unsplit_schedules(schedule, graph):
    """The stack API with R compute lanes under the policies that keep AT unsplit
    (FLOWMOE_AR, PIPE_MOE: all T rows of a block's input on lane 0, written chunk-wise on
    the lanes by the previous block) and FLOWMOE_AT: bit-identical to per-block calls of
    the default schedule on one lane (P = 1: the policies change only the schedule).
    Repeated three times to give a missing cross-lane dependency a chance to show."""
    from tests.gpu_util import run_stack_gpu
    cfg = CASES["c2_bench"]
    L = 3
    reps = [gen_replicated(cfg, block=l) for l in range(L)]
    wk = gen_worker(cfg, 0)
    wk["forced"] = None
    ref = run_stack_gpu(cfg, reps, wk, compute_streams=1, api="per_block")
    for _ in range(3):
        g = run_stack_gpu(cfg, reps, wk, compute_streams=cfg.R, graph=graph, api="stack", schedule=schedule)
        for n in ("y", "dx"):
            assert np.array_equal(g[n], ref[n]), n
        for l in range(L):
            assert np.array_equal(g["grad_flat"][l], ref["grad_flat"][l]), l
            assert np.array_equal(g["dw1"][l], ref["dw1"][l]), l


@pytest.mark.parametrize("dtype,graph", [("bf16", False), ("bf16", True), ("float32", False), ("tok", True)])
def test_stack_api_matches_per_block(dtype, graph):
    """flowmoe_stack_fwd/bwd (lanes forked once, chunks chained across blocks) gives
    bit-identical activations and grads to L block_fwd/block_bwd calls: the same kernels
    run on the same lane per chunk, only the block-boundary joins are gone."""
    from tests.gpu_util import run_stack_gpu
    cfg = {"bf16": CASES["c2_bench"], "tok": TOK_CASES["tok_bf16_dh128_r8"]}.get(
        dtype, CASES["c1_f32"].replace(R=4, residual=1, causal=1))
    L = 3
    reps = [gen_replicated(cfg, block=l) for l in range(L)]
    wk = gen_worker(cfg, 0)
    wk["forced"] = None
    ref = run_stack_gpu(cfg, reps, wk, compute_streams=cfg.R, api="per_block")
    g = run_stack_gpu(cfg, reps, wk, compute_streams=cfg.R, graph=graph, api="stack")
    for n in ("y", "dx"):
        assert np.array_equal(g[n], ref[n]), n
    for l in range(L):
        assert np.array_equal(g["grad_flat"][l], ref["grad_flat"][l]), l
        assert np.array_equal(g["dw1"][l], ref["dw1"][l]), l


# --------------------------------------------------------------- optimizer (reading Q17)
@pytest.mark.parametrize("kind", ["sgd", "adamw"])
def test_optimizer_step_matches_oracle(kind):
    """Three steps on a ragged-length tensor (vector + scalar tail) and on an unaligned
    view (scalar path): fp32 master/state vs the fp64 definitions, and the bf16 compute
    copy equals bf16(master)."""
    import torch
    from oracle.optim import adamw_step, sgd_momentum_step
    dev = torch.device("cuda", 0)
    ctx = fm.FlowMoE(fm.BlockShape(B=128, seq_len=64, M=64, n_heads=1, E=4, top_k=2, d_ffn=64, R=2,
                                   dtype="bf16"), 0, None)
    hp = dict(lr=3e-2, beta1=0.9, beta2=0.99, eps=1e-6, weight_decay=0.05)
    opt = fm.Optimizer.make(kind, **hp)
    rng = np.random.default_rng(5)
    for n, off in ((4099, 0), (1000, 1)):
        w0 = rng.standard_normal(n + off)
        buf = torch.tensor(w0, dtype=torch.float32, device=dev)
        master = buf[off:]
        s1 = torch.zeros(n + off, dtype=torch.float32, device=dev)[off:]
        s2 = torch.zeros(n + off, dtype=torch.float32, device=dev)[off:]
        wb = torch.empty(n, dtype=torch.bfloat16, device=dev)
        w, a, b = w0[off:].astype(np.float32).astype(np.float64), np.zeros(n), np.zeros(n)
        for step in (1, 2, 3):
            g = rng.standard_normal(n).astype(np.float32)
            gt = torch.tensor(g, device=dev)
            ctx.optimizer_step(opt, step, master, s1, s2 if kind == "adamw" else None, gt, wb)
            if kind == "adamw":
                w, a, b = adamw_step(w, a, b, g, step=step, **hp)
            else:
                w, a = sgd_momentum_step(w, a, g, lr=hp["lr"], momentum=hp["beta1"],
                                         weight_decay=hp["weight_decay"], step=step)
        torch.cuda.synchronize()
        got = master.cpu().numpy().astype(np.float64)
        assert rel(got, w) <= 1e-5, (n, off)
        assert rel(s1.cpu().numpy().astype(np.float64), a) <= 1e-5
        assert torch.equal(wb, master.to(torch.bfloat16))
    ctx.close()


def test_expert_update_behind_backward():
    """the expert update enqueued after a block's backward runs behind that block's
    expert wgrads and updates the master and the compute copy the next forward reads."""
    import torch
    from oracle.optim import adamw_step
    cfg = CASES["bf16_small"]
    rep = gen_replicated(cfg)
    wk = gen_worker(cfg, 0)
    dev = torch.device("cuda", 0)
    from tests.gpu_util import shape_of
    ctx = fm.FlowMoE(shape_of(cfg, 1, 0, "overwrite", cfg.R, "flowmoe"), 0, None)
    bt = fm.BlockTensors(rep, cfg.dtype, 0, 1, dev)
    names = ("w1", "b1", "w2", "b2")
    master = {n: bt.t[n].float().clone() for n in names}
    m = {n: torch.zeros_like(master[n]) for n in names}
    v = {n: torch.zeros_like(master[n]) for n in names}
    st = fm.ExpertOpt((ctypes.c_void_p * 4)(*[master[n].data_ptr() for n in names]),
                      (ctypes.c_void_p * 4)(*[m[n].data_ptr() for n in names]),
                      (ctypes.c_void_p * 4)(*[v[n].data_ptr() for n in names]),
                      (ctypes.c_void_p * 4)(*[bt.t[n].data_ptr() for n in names]))
    hp = dict(lr=1e-2, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)
    opt = fm.Optimizer.make("adamw", **hp)
    x = fm.to_device(wk["x"], cfg.dtype, dev)
    dy = fm.to_device(wk["dy"], cfg.dtype, dev)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    saved = torch.empty(ctx.saved_bytes, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()
    w_before = {n: master[n].double().cpu().numpy() for n in names}
    ctx.block_fwd(bt.params, x, y, saved, s)
    t = ctx.block_bwd(bt.params, x, saved, dy, dx, bt.grads, 1 << 20, s)
    tu = ctx.expert_update(opt, 1, st, bt.grads)
    ctx.allreduce_wait(t, s)
    ctx.allreduce_wait(tu, s)
    torch.cuda.synchronize()
    gname = {"w1": "dw1", "b1": "db1", "w2": "dw2", "b2": "db2"}
    for n in names:
        g = bt.g[gname[n]].double().cpu().numpy()
        assert np.abs(g).max() > 0, n  # the grads were final when the update ran
        want, _, _ = adamw_step(w_before[n], 0.0, 0.0, g, step=1, **hp)
        assert rel(master[n].double().cpu().numpy(), want) <= 1e-5, n
        assert torch.equal(bt.t[n], master[n].to(torch.bfloat16)), n
    ctx.close()


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_embedding_and_xent_vs_oracle(dtype):
    """Model edges through the C ABI: embedding gather (exact), its deterministic
    scatter-add (several id tiles, repeated and out-of-range ids, accumulate mode) and
    the softmax cross-entropy (ignored rows, ragged V) against oracle/model.py."""
    import torch
    from oracle.model import embed_backward, embed_forward, xent
    from tests.gpu_util import shape_of
    cfg = CASES["c1_f32"] if dtype == "f32" else CASES["bf16_small"]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ctx = fm.FlowMoE(shape_of(cfg, 1, 0), 0, None)
    rng = np.random.default_rng(21)
    V, T, M = 1000, 3000, cfg.M
    table = fm.to_device(rng.standard_normal((V, M)), dtype, dev)
    ids_h = rng.integers(0, V, T).astype(np.int32)
    ids_h[rng.integers(0, T, 40)] = 17          # a hot row
    ids_h[[5, 2999]] = [-1, V + 3]              # out of range: zero rows, no gradient
    ids = torch.from_numpy(ids_h).to(dev)
    x = torch.empty((T, M), dtype=fm.torch_dtype(dtype), device=dev)
    ctx.embed_fwd(table, ids, x)
    dx = fm.to_device(rng.standard_normal((T, M)), dtype, dev)
    dtab = torch.full((V, M), 0.5, dtype=torch.float32, device=dev)
    ctx.embed_bwd(ids, dx, dtab)
    Vx, T2 = 5000, 300
    lg_h = rng.standard_normal((T2, Vx)) * 3
    lab_h = rng.integers(0, Vx, T2).astype(np.int32)
    lab_h[[0, 7, 299]] = -1
    lg = torch.from_numpy(lg_h.astype(np.float32)).to(dev)
    lab = torch.from_numpy(lab_h).to(dev)
    losses = torch.empty(T2, dtype=torch.float32, device=dev)
    loss = torch.empty(1, dtype=torch.float32, device=dev)
    dl = torch.empty((T2, Vx), dtype=fm.torch_dtype(dtype), device=dev)
    ctx.xent(lg, lab, 1.0 / T2, losses, loss, dl)
    torch.cuda.synchronize()
    ctx.close()
    tab_h = fm.to_host_f64(table)
    assert np.array_equal(fm.to_host_f64(x), embed_forward(tab_h, ids_h))
    ref = embed_backward(ids_h, fm.to_host_f64(dx), V)
    assert rel(dtab.cpu().numpy().astype(np.float64) - 0.5, ref) <= 1e-5
    rl, rloss, rdl = xent(lg.cpu().numpy().astype(np.float64), lab_h, 1.0 / T2)
    assert rel(losses.cpu().numpy().astype(np.float64), rl) <= 1e-5
    assert abs(float(loss.item()) - rloss) <= 1e-5 * abs(rloss)
    assert rel(fm.to_host_f64(dl), rdl) <= (1e-5 if dtype == "f32" else 1e-2)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_lm_head_and_loss_chain_vs_oracle(dtype):
    """h -> logits (LM head) -> cross-entropy -> dlogits -> dh, dW through the C ABI,
    against oracle/model.py on the same device-rounded inputs (ragged T, V = 5000)."""
    import torch
    from oracle.model import lm_head_backward, lm_head_forward, xent
    from tests.gpu_util import shape_of
    cfg = CASES["c1_f32"] if dtype == "f32" else CASES["bf16_small"]
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    ctx = fm.FlowMoE(shape_of(cfg, 1, 0), 0, None)
    rng = np.random.default_rng(33)
    T, V, M = 300, 5000, cfg.M
    h = fm.to_device(rng.standard_normal((T, M)), dtype, dev)
    w = fm.to_device(rng.standard_normal((V, M)) / np.sqrt(M), dtype, dev)
    lab = torch.from_numpy(rng.integers(0, V, T).astype(np.int32)).to(dev)
    f32 = dict(dtype=torch.float32, device=dev)
    logits = torch.empty((T, V), **f32)
    ctx.lm_head_fwd(h, w, logits)
    losses, loss = torch.empty(T, **f32), torch.empty(1, **f32)
    dl = torch.empty((T, V), dtype=fm.torch_dtype(dtype), device=dev)
    ctx.xent(logits, lab, 1.0 / T, losses, loss, dl)
    dh = torch.empty((T, M), dtype=fm.torch_dtype(dtype), device=dev)
    dw = torch.full((V, M), 0.25, **f32)
    ctx.lm_head_bwd(h, w, dl, dh, dw)
    torch.cuda.synchronize()
    ctx.close()
    tol = TOL[dtype]
    hh, wh, dlh = fm.to_host_f64(h), fm.to_host_f64(w), fm.to_host_f64(dl)
    assert rel(logits.cpu().numpy().astype(np.float64), lm_head_forward(hh, wh)) <= (1e-5 if dtype == "f32" else 1e-3)
    _, rloss, _ = xent(logits.cpu().numpy().astype(np.float64), lab.cpu().numpy(), 1.0 / T)
    assert abs(float(loss.item()) - rloss) <= 1e-5 * abs(rloss)
    rdh, rdw = lm_head_backward(hh, wh, dlh)
    assert rel(fm.to_host_f64(dh), rdh) <= tol
    assert rel(dw.cpu().numpy().astype(np.float64) - 0.25, rdw) <= (1e-4 if dtype == "f32" else 1e-3)
