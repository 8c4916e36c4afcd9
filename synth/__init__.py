"""Seeded synthetic inputs for the FlowMoE block hot path.

This module is the ONLY code shared by the oracle (``oracle/``) and the CUDA path
(``paper_2510_00207_b200``).  It draws random numbers and rounds them to the
storage dtype; it holds none of the method's arithmetic (no capacity formula,
no routing, no softmax, no GEMM).  Random numbers the method would draw do not
exist (FlowMoE routing is deterministic), so only inputs come from here.

Workload recipe:
  X ~ N(0,1); Wq,Wk,Wv,Wo,Wg,W1 ~ N(0, 1/M); W2 ~ N(0, 1/F); b1,b2 ~ N(0, 0.02^2);
  dO ~ N(0,1).  Routing is balanced by default (i.i.d. Gaussian gate); the
  ``skew`` option adds a rank-1 Zipf(s=1) preference u·alpha^T to Wg and c·u to
  X so that expert popularity follows Zipf and capacity drops occur
  (P:1355 studies f-driven imbalance).
Seeds: numpy PCG64 seeded by SeedSequence([base, block, rank, stream]).
Replicated tensors (MHA, gate, all E experts) use rank = -1 -> 0xFFFF so every
worker sees the same weights; per-worker tensors (X, dO, forced routing) use
the worker rank.
"""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass

import numpy as np

SEED_BASE = 20251000
_REPL = 0xFFFF


@dataclass(frozen=True)
class BlockConfig:
    """Shapes of one FlowMoE block on one worker (names per SURVEY.md §0).

    T: tokens per worker (paper B·N), seq_len: N, M: model dim, n_heads: h,
    E: experts, top_k: k, d_ffn: F (paper H), R: pipelining degree,
    capacity_factor: f (0 = dropless), P: world size.
    """
    T: int
    seq_len: int
    M: int
    n_heads: int
    E: int
    top_k: int
    d_ffn: int
    R: int
    capacity_factor: float = 1.0
    causal: int = 0
    residual: int = 0
    P: int = 1
    dtype: str = "bf16"  # "f32" or "bf16" (storage of activations/weights)

    def replace(self, **kw) -> "BlockConfig":
        return dataclasses.replace(self, **kw)


# SURVEY.md §8(d) configs restated as concrete synthetic shapes.
PRESETS = {
    # configs[0]: fp32, 256 tokens, M=64, 4 heads, E=4 top-2, F=128, R=2, 2 workers
    "c1": BlockConfig(T=256, seq_len=64, M=64, n_heads=4, E=4, top_k=2, d_ffn=128, R=2,
                      capacity_factor=1.0, causal=0, residual=0, P=2, dtype="f32"),
    "c1_dropless": BlockConfig(T=256, seq_len=64, M=64, n_heads=4, E=4, top_k=2, d_ffn=128, R=2,
                               capacity_factor=0.0, causal=0, residual=0, P=2, dtype="f32"),
    # configs[1]: GPT2-Tiny-MoE-shaped (Table 3: L=12, B=4, N=256, M=256, H=512, k=2, f=1.0), E=8
    "c2": BlockConfig(T=1024, seq_len=256, M=256, n_heads=4, E=8, top_k=2, d_ffn=512, R=4,
                      capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    # configs[2]: BERT-Large-MoE-shaped (M=1024, 16 heads, E=16, top-2), F=2048, T=4x512
    "c3": BlockConfig(T=2048, seq_len=512, M=1024, n_heads=16, E=16, top_k=2, d_ffn=2048, R=2,
                      capacity_factor=1.0, causal=0, residual=1, P=1, dtype="bf16"),
    # configs[3]: LLaMA2-MoE-shaped (M=4096, 32 heads, E=16, top-2), F=16384, T=4x512
    "c4": BlockConfig(T=2048, seq_len=512, M=4096, n_heads=32, E=16, top_k=2, d_ffn=16384, R=2,
                      capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
    # configs[4] point: DeepSeek-V2-S-shaped fine-grained experts (M=5120, F=1536, k=8), E=16
    "dsv2s": BlockConfig(T=1024, seq_len=256, M=5120, n_heads=40, E=16, top_k=8, d_ffn=1536, R=2,
                         capacity_factor=1.0, causal=1, residual=1, P=1, dtype="bf16"),
}


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round to the nearest bfloat16 (ties to even), returned as float64.

    Storage-dtype conversion of an input, identical to what the device holds
    after a host->device copy of the bf16 bits returned by ``bf16_bits``.
    """
    bits = bf16_bits(a)
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """uint16 bfloat16 bit patterns of ``a`` (round-to-nearest-even via fp32)."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float32))
    u = f.view(np.uint32).astype(np.uint64)
    rounding = ((u >> 16) & 1) + 0x7FFF
    out = ((u + rounding) >> 16).astype(np.uint16)
    # NaN stays NaN (never produced by this generator, kept for completeness)
    nan = np.isnan(f)
    if nan.any():
        out[nan] = 0x7FC0
    return out


def storage_round(a: np.ndarray, dtype: str) -> np.ndarray:
    """Round an fp64 array to the storage dtype and return it as fp64."""
    if dtype == "bf16":
        return bf16_round(a)
    if dtype == "f32":
        return np.asarray(a, dtype=np.float32).astype(np.float64)
    raise ValueError(dtype)


def _rng(block: int, rank: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(
        np.random.SeedSequence([SEED_BASE, block, rank & 0xFFFF, stream])))


def gen_replicated(cfg: BlockConfig, block: int = 0, skew: bool = False) -> dict:
    """Weights shared by all workers: MHA, gate and all E experts (fp64, storage-rounded)."""
    M, E, F = cfg.M, cfg.E, cfg.d_ffn
    r = _rng(block, _REPL, 1)
    out = {
        "wqkv": r.standard_normal((M, 3 * M)) / np.sqrt(M),
        "wo": r.standard_normal((M, M)) / np.sqrt(M),
        "wg": r.standard_normal((M, E)) / np.sqrt(M),
        "w1": r.standard_normal((E, M, F)) / np.sqrt(M),
        "b1": 0.02 * r.standard_normal((E, F)),
        "w2": r.standard_normal((E, F, M)) / np.sqrt(F),
        "b2": 0.02 * r.standard_normal((E, M)),
    }
    if skew:
        u = _rng(block, _REPL, 7).standard_normal(M)
        u /= np.linalg.norm(u)
        zipf = 1.0 / np.arange(1, E + 1)
        alpha = np.log(zipf / zipf.sum())
        out["wg"] = out["wg"] + np.outer(u, alpha - alpha.mean())
    return {k: storage_round(v, cfg.dtype) for k, v in out.items()}


def gen_worker(cfg: BlockConfig, rank: int = 0, block: int = 0, skew: bool = False) -> dict:
    """Per-worker tensors: X [T,M], dO [T,M] (storage-rounded fp64) and a forced
    routing ``forced_idx`` [T,k] int32 of k distinct experts per token."""
    T, M, E, k = cfg.T, cfg.M, cfg.E, cfg.top_k
    r = _rng(block, rank, 2)
    x = r.standard_normal((T, M))
    if skew:
        u = _rng(block, _REPL, 7).standard_normal(M)
        u /= np.linalg.norm(u)
        x = x + 4.0 * u[None, :]
    d_o = _rng(block, rank, 3).standard_normal((T, M))
    keys = _rng(block, rank, 4).random((T, E))
    forced = np.argsort(keys, axis=1, kind="stable")[:, :k].astype(np.int32)
    return {"x": storage_round(x, cfg.dtype), "dy": storage_round(d_o, cfg.dtype),
            "forced_idx": forced}


def to_device_dtype(a: np.ndarray, dtype: str) -> np.ndarray:
    """Host array in the device storage format: uint16 bf16 bits or float32."""
    if dtype == "bf16":
        return bf16_bits(a)
    return np.asarray(a, dtype=np.float32)


def gen_device_block(cfg: BlockConfig, rank: int, P: int, block: int, device):
    """Device-side weights of one block for rank ``rank`` of ``P`` (local experts
    only), same distributions as gen_replicated, drawn with a seeded torch
    generator on the device.  Used by bench.py, where full-size configs are too
    large for host fp64 generation; parity tests use gen_replicated."""
    import torch
    M, E, F = cfg.M, cfg.E, cfg.d_ffn
    El = E // P
    g = torch.Generator(device=device)
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32

    def randn(shape, std, stream):
        g.manual_seed(SEED_BASE * 1000003 + block * 7919 + stream)
        return (torch.randn(shape, generator=g, device=device, dtype=torch.float32) * std).to(dt)

    out = {"wqkv": randn((M, 3 * M), M ** -0.5, 1), "wo": randn((M, M), M ** -0.5, 2),
           "wg": randn((M, E), M ** -0.5, 3)}
    w1, b1, w2, b2 = [], [], [], []
    for el in range(El):
        e = rank * El + el
        w1.append(randn((M, F), M ** -0.5, 100 + 4 * e))
        b1.append(randn((F,), 0.02, 101 + 4 * e))
        w2.append(randn((F, M), F ** -0.5, 102 + 4 * e))
        b2.append(randn((M,), 0.02, 103 + 4 * e))
    out.update(w1=torch.stack(w1), b1=torch.stack(b1), w2=torch.stack(w2), b2=torch.stack(b2))
    return out


def gen_device_worker(cfg: BlockConfig, rank: int, device):
    """Device-side X [T,M] and dO [T,M] ~ N(0,1) for rank ``rank``."""
    import torch
    g = torch.Generator(device=device)
    dt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    g.manual_seed(SEED_BASE * 31 + 2 * rank + 1)
    x = torch.randn((cfg.T, cfg.M), generator=g, device=device).to(dt)
    g.manual_seed(SEED_BASE * 31 + 2 * rank + 2)
    dy = torch.randn((cfg.T, cfg.M), generator=g, device=device).to(dt)
    return x, dy
