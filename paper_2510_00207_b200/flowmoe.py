"""Thin ctypes binding of libflowmoe.so (include/flowmoe.h).

Argument marshalling only: every step of the block runs in the library's CUDA
kernels.  PyTorch provides device memory, streams and process groups.  There is
no fallback: if the shared library is missing or fails to load, importing the
binding raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# FLOWMOE_LIB: load another build of the same ABI (A/B measurements of kernel changes)
LIB_PATH = os.environ.get("FLOWMOE_LIB") or os.path.join(_HERE, "libflowmoe.so")

FLOWMOE_F32, FLOWMOE_BF16 = 0, 1
SCHEDULES = {"flowmoe": 0, "flowmoe_ar": 1, "flowmoe_at": 2, "pipe_moe": 3, "vanilla_ep": 4}

# include/flowmoe.h (product ABI) and include/flowmoe_test.h (test / benchmark hooks)
EXPORTED = [
    "flowmoe_get_unique_id", "flowmoe_create", "flowmoe_saved_bytes", "flowmoe_grad_flat_count",
    "flowmoe_block_fwd", "flowmoe_block_bwd", "flowmoe_stack_fwd", "flowmoe_stack_bwd", "flowmoe_allreduce_submit",
    "flowmoe_allreduce_wait", "flowmoe_register_saved", "flowmoe_unregister_saved", "flowmoe_check_health",
    "flowmoe_optimizer_step", "flowmoe_expert_update", "flowmoe_embed_fwd", "flowmoe_embed_bwd", "flowmoe_xent",
    "flowmoe_lm_head_fwd", "flowmoe_lm_head_bwd", "flowmoe_set_forced_routing",
    "flowmoe_status_string", "flowmoe_last_error", "flowmoe_destroy",
]
EXPORTED_TEST = [
    "flowmoe_saved_routing_offsets", "flowmoe_debug_set", "flowmoe_test_gemm", "flowmoe_profile_begin",
    "flowmoe_profile_end", "flowmoe_kernel_launches", "flowmoe_create_local_group", "flowmoe_test_arrivals",
    "flowmoe_tasklog_begin", "flowmoe_tasklog_end", "flowmoe_test_exchange",
]
TASK_KINDS = ("AT", "D", "E", "C", "MERGE", "CBPACK", "CB", "EB", "DB", "WGE", "ATB", "WGA", "AR")


class FlowMoEError(RuntimeError):
    pass


class Config(ctypes.Structure):
    _fields_ = [("B", ctypes.c_int64), ("seq_len", ctypes.c_int32), ("M", ctypes.c_int32),
                ("n_heads", ctypes.c_int32), ("E", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("d_ffn", ctypes.c_int32), ("R", ctypes.c_int32),
                ("capacity_factor", ctypes.c_float), ("causal", ctypes.c_int32),
                ("residual", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("world_size", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("grad_mode", ctypes.c_int32), ("compute_streams", ctypes.c_int32),
                ("schedule", ctypes.c_int32), ("a2a_impl", ctypes.c_int32)]


class ProfEntry(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char_p), ("launches", ctypes.c_int64), ("ms", ctypes.c_double),
                ("flops", ctypes.c_double), ("bytes", ctypes.c_double)]


class TaskRec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("block", ctypes.c_int32), ("chunk", ctypes.c_int32),
                ("dir", ctypes.c_int32), ("stream", ctypes.c_uint64), ("t0_ms", ctypes.c_double),
                ("t1_ms", ctypes.c_double)]


class Params(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("wqkv", "wo", "wg", "w1", "b1", "w2", "b2")]


class Grads(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("grad_flat", "dw1", "db1", "dw2", "db2")]


OPT_KINDS = {"sgd": 0, "adamw": 1}


class Optimizer(ctypes.Structure):
    """flowmoe_optimizer: kind ('sgd' momentum / 'adamw'), lr, beta1 (SGD momentum), beta2, eps,
    weight_decay."""
    _fields_ = [("kind", ctypes.c_int32), ("lr", ctypes.c_float), ("beta1", ctypes.c_float),
                ("beta2", ctypes.c_float), ("eps", ctypes.c_float), ("weight_decay", ctypes.c_float)]

    @classmethod
    def make(cls, kind="adamw", lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0):
        return cls(OPT_KINDS[kind], lr, beta1, beta2, eps, weight_decay)


class ExpertOpt(ctypes.Structure):
    """flowmoe_expert_opt: per tensor (w1, b1, w2, b2) fp32 master, state1, state2, compute copy."""
    _fields_ = [("master", ctypes.c_void_p * 4), ("state1", ctypes.c_void_p * 4),
                ("state2", ctypes.c_void_p * 4), ("weight", ctypes.c_void_p * 4)]


_lib = None


def lib() -> ctypes.CDLL:
    """Load libflowmoe.so (built by paper_2510_00207_b200.build / __graft_entry__.build)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise FlowMoEError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    vp, sz, i32, u64, i64 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64
    L.flowmoe_get_unique_id.argtypes = [ctypes.c_char_p]
    L.flowmoe_create.argtypes = [ctypes.POINTER(Config), ctypes.c_char_p, i32, ctypes.POINTER(vp)]
    L.flowmoe_saved_bytes.argtypes = [vp]
    L.flowmoe_saved_bytes.restype = sz
    L.flowmoe_grad_flat_count.argtypes = [vp]
    L.flowmoe_grad_flat_count.restype = sz
    L.flowmoe_block_fwd.argtypes = [vp, ctypes.POINTER(Params), vp, vp, vp, vp]
    L.flowmoe_block_bwd.argtypes = [vp, ctypes.POINTER(Params), vp, vp, vp, vp,
                                    ctypes.POINTER(Grads), sz, ctypes.POINTER(u64), vp]
    L.flowmoe_stack_fwd.argtypes = [vp, i32, ctypes.POINTER(Params), vp, ctypes.POINTER(vp),
                                    ctypes.POINTER(vp), vp]
    L.flowmoe_stack_bwd.argtypes = [vp, i32, ctypes.POINTER(Params), vp, ctypes.POINTER(vp),
                                    ctypes.POINTER(vp), vp, ctypes.POINTER(vp), ctypes.POINTER(Grads), sz,
                                    ctypes.POINTER(u64), vp]
    L.flowmoe_optimizer_step.argtypes = [vp, ctypes.POINTER(Optimizer), ctypes.c_int64, vp, vp, vp, vp, vp, sz, vp]
    L.flowmoe_expert_update.argtypes = [vp, ctypes.POINTER(Optimizer), ctypes.c_int64, ctypes.POINTER(ExpertOpt),
                                        ctypes.POINTER(Grads), ctypes.POINTER(u64)]
    L.flowmoe_embed_fwd.argtypes = [vp, vp, i64, vp, i64, vp, vp]
    L.flowmoe_embed_bwd.argtypes = [vp, vp, i64, vp, i64, vp, vp]
    L.flowmoe_xent.argtypes = [vp, vp, vp, i64, i64, ctypes.c_float, vp, vp, vp, vp]
    L.flowmoe_lm_head_fwd.argtypes = [vp, vp, vp, i64, i64, vp, vp]
    L.flowmoe_lm_head_bwd.argtypes = [vp, vp, vp, vp, i64, i64, vp, vp, vp]
    L.flowmoe_allreduce_submit.argtypes = [vp, vp, sz, sz, i32, vp, ctypes.POINTER(u64)]
    L.flowmoe_allreduce_wait.argtypes = [vp, u64, vp]
    L.flowmoe_register_saved.argtypes = [vp, vp]
    L.flowmoe_unregister_saved.argtypes = [vp, vp]
    L.flowmoe_check_health.argtypes = [vp]
    L.flowmoe_test_arrivals.argtypes = [vp, ctypes.POINTER(ctypes.c_uint), sz]
    L.flowmoe_test_exchange.argtypes = [vp, vp, i32, i32, i32, vp]
    L.flowmoe_create_local_group.argtypes = [ctypes.POINTER(Config), i32, i32, ctypes.POINTER(vp)]
    L.flowmoe_set_forced_routing.argtypes = [vp, vp]
    L.flowmoe_saved_routing_offsets.argtypes = [vp] + [ctypes.POINTER(sz)] * 5
    L.flowmoe_debug_set.argtypes = [vp, i32, i32]
    L.flowmoe_kernel_launches.restype = u64
    L.flowmoe_test_gemm.argtypes = [vp, i32, i32, i32, i32, i32, vp, i64, i64, i32, vp, i64, i64, i32,
                                    vp, i64, i64, i32, vp, vp, vp, vp]
    L.flowmoe_profile_begin.argtypes = [vp]
    L.flowmoe_tasklog_begin.argtypes = [vp]
    L.flowmoe_tasklog_end.argtypes = [vp, ctypes.POINTER(TaskRec), i32]
    L.flowmoe_tasklog_end.restype = i32
    L.flowmoe_profile_end.argtypes = [vp, ctypes.POINTER(ProfEntry), i32]
    L.flowmoe_profile_end.restype = i32
    L.flowmoe_status_string.argtypes = [i32]
    L.flowmoe_status_string.restype = ctypes.c_char_p
    L.flowmoe_last_error.restype = ctypes.c_char_p
    L.flowmoe_destroy.argtypes = [vp]
    L.flowmoe_destroy.restype = None
    _lib = L
    return L


# environment knobs applied to every ctx at creation (flowmoe_test.h flowmoe_debug_set)
_ENV_KNOBS = (("FLOWMOE_DEBUG_SIMT", 1, 1),        # debug: route bf16 GEMMs to the SIMT kernel
              ("FLOWMOE_DEBUG_SWAP", 2, 1),        # debug: swap MN-major descriptor strides
              ("FLOWMOE_DEBUG_SIMT_ATTN", 3, 1),   # debug: SIMT attention for bf16
              ("FLOWMOE_NO_PDL", 4, 0),            # A/B: plain stream-ordered launches
              ("FLOWMOE_P2P_A2A_STREAM", 6, 0),    # A/B: peer-memory A2A on the A2A stream
              ("FLOWMOE_FORCE_CG1", 7, 1),         # A/B: single-CTA GEMM tiles only
              ("FLOWMOE_FORCE_CG2", 7, 2),         # test: CTA-pair (cta_group::2) GEMMs everywhere
              ("FLOWMOE_NO_STREAMK", 8, 1))        # A/B: whole-tile GEMM work split only
_ENV_VALUE_KNOBS = (("FLOWMOE_BWD_SM_RESERVE", 9),  # A/B: SMs the backward GEMMs leave to the AR (P > 1)
                    ("FLOWMOE_SM_RESERVE", 10))     # A/B: SMs every GEMM leaves to the other lanes


def _apply_env_knobs(handle):
    for env, key, val in _ENV_KNOBS:
        if os.environ.get(env):
            _check(lib().flowmoe_debug_set(handle, key, val), "flowmoe_debug_set")
    for env, key in _ENV_VALUE_KNOBS:
        if os.environ.get(env):
            _check(lib().flowmoe_debug_set(handle, key, int(os.environ[env])), "flowmoe_debug_set")


def _check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise FlowMoEError(f"{what}: {L.flowmoe_status_string(rc).decode()} "
                           f"({L.flowmoe_last_error().decode()})")


def get_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().flowmoe_get_unique_id(buf), "flowmoe_get_unique_id")
    return buf.raw


def kernel_launches() -> int:
    return int(lib().flowmoe_kernel_launches())


def test_gemm(dtype: str, A, B, C, *, M, N, K, batch=1, lda, sA=0, a_mmajor=0, ldb, sB=0,
              b_kmajor=0, ldc, sC=0, epi=0, bias=None, resid=None, aux=None, stream=None, ctx=None):
    """One GEMM through the library's GEMM kernels (include/flowmoe_test.h flowmoe_test_gemm)."""
    _check(lib().flowmoe_test_gemm(ctx.handle if ctx is not None else None, FLOWMOE_BF16 if dtype == "bf16" else FLOWMOE_F32, M, N, K, batch,
                                   _ptr(A), lda, sA, a_mmajor, _ptr(B), ldb, sB, b_kmajor, _ptr(C),
                                   ldc, sC, epi, _ptr(bias), _ptr(resid), _ptr(aux),
                                   _stream_handle(stream)), "flowmoe_test_gemm")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_handle(stream):
    return ctypes.c_void_p(stream.cuda_stream if stream is not None else 0)


@dataclass
class BlockShape:
    """Config fields of one rank (mirrors flowmoe_config)."""
    B: int
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
    dtype: str = "bf16"
    world_size: int = 1
    rank: int = 0
    grad_mode: str = "accumulate"  # or "overwrite"
    compute_streams: int = 1
    schedule: str = "flowmoe"
    a2a_impl: str = "nccl"  # or "p2p"

    def to_c(self) -> Config:
        return Config(self.B, self.seq_len, self.M, self.n_heads, self.E, self.top_k, self.d_ffn,
                      self.R, self.capacity_factor, self.causal, self.residual,
                      FLOWMOE_BF16 if self.dtype == "bf16" else FLOWMOE_F32, self.world_size,
                      self.rank, 1 if self.grad_mode == "overwrite" else 0, self.compute_streams,
                      SCHEDULES[self.schedule], 1 if self.a2a_impl == "p2p" else 0)


class FlowMoE:
    """One FlowMoE context (one rank): flowmoe_create ... flowmoe_destroy."""

    def __init__(self, shape: BlockShape, device: int = 0, unique_id: bytes | None = None, _handle=None):
        L = lib()
        self.shape = shape
        self._cfg = shape.to_c()
        if _handle is None:
            h = ctypes.c_void_p()
            _check(L.flowmoe_create(ctypes.byref(self._cfg), unique_id, device, ctypes.byref(h)),
                   "flowmoe_create")
        else:
            h = _handle
        self.handle = h
        _apply_env_knobs(h)
        self.saved_bytes = int(L.flowmoe_saved_bytes(h))
        self.grad_flat_count = int(L.flowmoe_grad_flat_count(h))

    @classmethod
    def local_group(cls, shape: BlockShape, P: int, device: int = 0) -> list:
        """P ctxs of world_size P on one device (flowmoe_test.h flowmoe_create_local_group):
        the simulated world of the one-GPU exchange tests."""
        import dataclasses
        cfg = dataclasses.replace(shape, world_size=P, rank=0, a2a_impl="p2p").to_c()
        hs = (ctypes.c_void_p * P)()
        _check(lib().flowmoe_create_local_group(ctypes.byref(cfg), P, device, hs), "flowmoe_create_local_group")
        return [cls(dataclasses.replace(shape, world_size=P, rank=q, a2a_impl="p2p"), device,
                    _handle=ctypes.c_void_p(hs[q])) for q in range(P)]

    def register_saved(self, saved):
        _check(lib().flowmoe_register_saved(self.handle, _ptr(saved)), "flowmoe_register_saved")

    def unregister_saved(self, saved):
        _check(lib().flowmoe_unregister_saved(self.handle, _ptr(saved)), "flowmoe_unregister_saved")

    def arrivals(self) -> np.ndarray:
        """Peer-memory A2A arrival counters [4 kinds][R][world_size] (flowmoe_test_arrivals)."""
        n = 4 * self.shape.R * self.shape.world_size
        buf = (ctypes.c_uint * n)()
        _check(lib().flowmoe_test_arrivals(self.handle, buf, n), "flowmoe_test_arrivals")
        return np.array(buf[:], dtype=np.int64).reshape(4, self.shape.R, self.shape.world_size)

    def test_exchange(self, saved, kind: int, r: int, iters: int, stream=None):
        """iters back-to-back A2A exchanges of chunk r (flowmoe_test.h flowmoe_test_exchange)."""
        _check(lib().flowmoe_test_exchange(self.handle, _ptr(saved), kind, r, iters, _stream_handle(stream)),
               "flowmoe_test_exchange")

    def check_health(self):
        _check(lib().flowmoe_check_health(self.handle), "flowmoe_check_health")

    def debug_set(self, key: int, value: int):
        _check(lib().flowmoe_debug_set(self.handle, key, value), "flowmoe_debug_set")

    def tasklog_begin(self):
        _check(lib().flowmoe_tasklog_begin(self.handle), "flowmoe_tasklog_begin")

    def tasklog_end(self, max_entries: int = 65536) -> list[dict]:
        """Measured task intervals since tasklog_begin (flowmoe_test.h flowmoe_tasklog_end)."""
        buf = (TaskRec * max_entries)()
        n = lib().flowmoe_tasklog_end(self.handle, buf, max_entries)
        if n < 0:
            raise FlowMoEError(f"flowmoe_tasklog_end: {lib().flowmoe_last_error().decode()}")
        return [dict(kind=TASK_KINDS[buf[i].kind], block=buf[i].block, chunk=buf[i].chunk, dir=buf[i].dir,
                     stream=buf[i].stream, t0=buf[i].t0_ms, t1=buf[i].t1_ms) for i in range(n)]

    def profile_begin(self):
        _check(lib().flowmoe_profile_begin(self.handle), "flowmoe_profile_begin")

    def profile_end(self) -> list[dict]:
        """Per-kernel-kind device time and algorithmic work since profile_begin()."""
        buf = (ProfEntry * 64)()
        n = lib().flowmoe_profile_end(self.handle, buf, 64)
        if n < 0:
            raise FlowMoEError(f"flowmoe_profile_end: {lib().flowmoe_last_error().decode()}")
        return [dict(name=buf[i].name.decode(), launches=buf[i].launches, ms=buf[i].ms,
                     flops=buf[i].flops, bytes=buf[i].bytes) for i in range(n)]

    def close(self):
        if getattr(self, "handle", None):
            lib().flowmoe_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def routing_offsets(self) -> dict:
        vals = [ctypes.c_size_t() for _ in range(5)]
        _check(lib().flowmoe_saved_routing_offsets(self.handle, *[ctypes.byref(v) for v in vals]),
               "flowmoe_saved_routing_offsets")
        return dict(zip(("logits", "idx", "w", "pos", "counts"), (v.value for v in vals)))

    def set_forced_routing(self, idx):
        _check(lib().flowmoe_set_forced_routing(self.handle, _ptr(idx)), "flowmoe_set_forced_routing")

    def block_fwd(self, params: Params, x, y, saved, stream=None):
        _check(lib().flowmoe_block_fwd(self.handle, ctypes.byref(params), _ptr(x), _ptr(y),
                                       _ptr(saved), _stream_handle(stream)), "flowmoe_block_fwd")

    def block_bwd(self, params: Params, x, saved, dy, dx, grads: Grads, chunk_bytes: int,
                  stream=None) -> int:
        t = ctypes.c_uint64()
        _check(lib().flowmoe_block_bwd(self.handle, ctypes.byref(params), _ptr(x), _ptr(saved),
                                       _ptr(dy), _ptr(dx), ctypes.byref(grads), chunk_bytes,
                                       ctypes.byref(t), _stream_handle(stream)),
               "flowmoe_block_bwd")
        return t.value

    def stack_fwd(self, params: list, x0, ys: list, saved: list, stream=None):
        L = len(params)
        pa = (Params * L)(*params)
        yv = (ctypes.c_void_p * L)(*[t.data_ptr() for t in ys])
        sv = (ctypes.c_void_p * L)(*[t.data_ptr() for t in saved])
        _check(lib().flowmoe_stack_fwd(self.handle, L, pa, _ptr(x0), yv, sv, _stream_handle(stream)),
               "flowmoe_stack_fwd")

    def stack_bwd(self, params: list, x0, ys: list, saved: list, dy, dxs: list, grads: list,
                  chunk_bytes: int, stream=None) -> list:
        L = len(params)
        pa = (Params * L)(*params)
        yv = (ctypes.c_void_p * L)(*[t.data_ptr() for t in ys])
        sv = (ctypes.c_void_p * L)(*[t.data_ptr() for t in saved])
        dv = (ctypes.c_void_p * L)(*[(t.data_ptr() if t is not None else None) for t in dxs])
        gv = (Grads * L)(*grads)
        tk = (ctypes.c_uint64 * L)()
        _check(lib().flowmoe_stack_bwd(self.handle, L, pa, _ptr(x0), yv, sv, _ptr(dy), dv, gv, chunk_bytes,
                                       tk, _stream_handle(stream)), "flowmoe_stack_bwd")
        return list(tk)

    def allreduce_submit(self, buf, count: int, chunk_bytes: int, priority: int = 1,
                         ready_event=None) -> int:
        t = ctypes.c_uint64()
        ev = ctypes.c_void_p(ready_event.cuda_event) if ready_event is not None else None
        _check(lib().flowmoe_allreduce_submit(self.handle, _ptr(buf), count, chunk_bytes, priority,
                                              ev, ctypes.byref(t)), "flowmoe_allreduce_submit")
        return t.value

    def allreduce_wait(self, ticket: int, stream=None):
        _check(lib().flowmoe_allreduce_wait(self.handle, ticket, _stream_handle(stream)),
               "flowmoe_allreduce_wait")

    def optimizer_step(self, opt: "Optimizer", step: int, master, state1, state2, grad, weight=None,
                       stream=None):
        """One optimizer step over a tensor (fp32 master / state / grad, optional compute copy)."""
        _check(lib().flowmoe_optimizer_step(self.handle, ctypes.byref(opt), step, _ptr(master), _ptr(state1),
                                            _ptr(state2), _ptr(grad), _ptr(weight), master.numel(),
                                            _stream_handle(stream)), "flowmoe_optimizer_step")

    def embed_fwd(self, table, ids, x, stream=None):
        """x[t] = table[ids[t]] (table [V][M], ids [T] int32, x [T][M], config dtype)."""
        _check(lib().flowmoe_embed_fwd(self.handle, _ptr(table), table.shape[0], _ptr(ids), ids.numel(), _ptr(x),
                                       _stream_handle(stream)), "flowmoe_embed_fwd")

    def embed_bwd(self, ids, dx, dtable, stream=None):
        """dtable[v] += sum of dx[t] over ids[t] == v (dtable fp32 [V][M], deterministic)."""
        _check(lib().flowmoe_embed_bwd(self.handle, _ptr(ids), ids.numel(), _ptr(dx), dtable.shape[0], _ptr(dtable),
                                       _stream_handle(stream)), "flowmoe_embed_bwd")

    def xent(self, logits, labels, scale: float, losses, loss=None, dlogits=None, stream=None):
        """Softmax cross-entropy of fp32 logits [T][V]: per-row losses, loss = scale·sum,
        dlogits = scale·(softmax - onehot) in the config dtype (rows with label < 0 ignored)."""
        T, V = logits.shape
        _check(lib().flowmoe_xent(self.handle, _ptr(logits), _ptr(labels), T, V, scale, _ptr(losses), _ptr(loss),
                                  _ptr(dlogits), _stream_handle(stream)), "flowmoe_xent")

    def lm_head_fwd(self, h, w, logits, stream=None):
        """logits [T][V] fp32 = h [T][M] · w [V][M]ᵀ."""
        _check(lib().flowmoe_lm_head_fwd(self.handle, _ptr(h), _ptr(w), h.shape[0], w.shape[0], _ptr(logits),
                                         _stream_handle(stream)), "flowmoe_lm_head_fwd")

    def lm_head_bwd(self, h, w, dlogits, dh=None, dw=None, stream=None):
        """dh = dlogits · w (overwritten), dw += dlogitsᵀ · h (fp32)."""
        _check(lib().flowmoe_lm_head_bwd(self.handle, _ptr(h), _ptr(w), _ptr(dlogits), dlogits.shape[0],
                                         dlogits.shape[1], _ptr(dh), _ptr(dw), _stream_handle(stream)),
               "flowmoe_lm_head_bwd")

    def expert_update(self, opt: "Optimizer", step: int, st: "ExpertOpt", grads: "Grads") -> int:
        """Expert update right behind the last enqueued backward's expert wgrads;
        returns a ticket for allreduce_wait."""
        t = ctypes.c_uint64(0)
        _check(lib().flowmoe_expert_update(self.handle, ctypes.byref(opt), step, ctypes.byref(st),
                                           ctypes.byref(grads), ctypes.byref(t)), "flowmoe_expert_update")
        return t.value


# ---------------------------------------------------------------- torch helpers
def torch_dtype(dtype: str):
    import torch
    return torch.bfloat16 if dtype == "bf16" else torch.float32


def to_device(a: np.ndarray, dtype: str, device):
    """Upload an fp64 host array as the device storage dtype (bf16 bits or fp32)."""
    import torch
    if dtype == "bf16":
        from synth import bf16_bits
        return torch.from_numpy(bf16_bits(a).view(np.int16)).to(device).view(torch.bfloat16)
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).to(device)


def to_host_f64(t) -> np.ndarray:
    import torch
    return t.detach().to(torch.float32).cpu().numpy().astype(np.float64)


class BlockTensors:
    """Device weights + grads of one block for rank `rank` of `P` (local experts only)."""

    def __init__(self, rep: dict, dtype: str, rank: int, P: int, device):
        import torch
        E = rep["w1"].shape[0]
        El = E // P
        sl = slice(rank * El, (rank + 1) * El)
        self.t = {
            "wqkv": to_device(rep["wqkv"], dtype, device), "wo": to_device(rep["wo"], dtype, device),
            "wg": to_device(rep["wg"], dtype, device), "w1": to_device(rep["w1"][sl], dtype, device),
            "b1": to_device(rep["b1"][sl], dtype, device), "w2": to_device(rep["w2"][sl], dtype, device),
            "b2": to_device(rep["b2"][sl], dtype, device),
        }
        M, F = rep["w1"].shape[1], rep["w1"].shape[2]
        f32 = dict(device=device, dtype=torch.float32)
        self.g = {
            "grad_flat": torch.zeros(4 * M * M + M * E, **f32),
            "dw1": torch.zeros(El, M, F, **f32), "db1": torch.zeros(El, F, **f32),
            "dw2": torch.zeros(El, F, M, **f32), "db2": torch.zeros(El, M, **f32),
        }
        self.params = Params(*[self.t[n].data_ptr() for n in ("wqkv", "wo", "wg", "w1", "b1", "w2", "b2")])
        self.grads = Grads(*[self.g[n].data_ptr() for n in ("grad_flat", "dw1", "db1", "dw2", "db2")])

    def zero_grads(self):
        for v in self.g.values():
            v.zero_()
