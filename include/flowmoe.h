/* flowmoe.h — C ABI of the B200-native FlowMoE block hot path (libflowmoe.so).
 *
 * What it computes: one training iteration of a transformer-MoE block —
 * MHA + top-k gating (task AT), A2A dispatch (D), expert FFN (E), A2A combine
 * (C), forward and backward — split into R micro-batch chunks and run as one
 * pipeline in the orders of Eqs.(3)-(6) (§3.2), with the
 * all-reduce of the replicated MHA and gating gradients (4M²+M·E parameters
 * per block) cut into S_p-byte chunks and issued at lower priority than
 * the A2A tasks (Alg. 2).  Block math: P:75-76 (MHA W^Q,W^K,
 * W^V,W^O ∈ R^{M×M}; gate = linear M×E + softmax + top-k; capacity
 * C = f·k·B·N/E; experts M×H then H×M).  Readings of points the paper leaves
 * open are listed in DESIGN.md ("Readings").
 *
 * Conventions
 *  - Row-vector convention y = x·W; every weight is stored [in][out] row-major.
 *  - "tokens" B (this ABI) = the paper's B·N on one rank; chunk r of R covers
 *    whole sequences [r·S/R, (r+1)·S/R) (reading Q1), S = B/seq_len.
 *  - dtype BF16: activations and weights bf16, fp32 accumulation, grads fp32.
 *    dtype F32: everything fp32 with true-fp32 (non-TF32) arithmetic.
 *  - All device pointers are CUDA device memory of the ctx's device; every
 *    enqueueing call is host-synchronous for validation and stream-ordered
 *    (asynchronous) for the work.  Nothing is enqueued when a call returns an
 *    error.  Nothing throws or aborts across the ABI.
 *  - Ownership: the caller owns x, y, dy, dx, params, grads and `saved`
 *    (sized by flowmoe_saved_bytes, one per block of a stack); pointers must
 *    stay valid until the enqueued work completes.  The ctx owns its streams,
 *    events, NCCL communicators and backward workspaces (reused across blocks).
 */
#ifndef FLOWMOE_H
#define FLOWMOE_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  FLOWMOE_OK = 0,
  FLOWMOE_ERR_INVALID = 1,     /* a config field or argument is invalid; message names it */
  FLOWMOE_ERR_CUDA = 2,        /* a CUDA runtime call or kernel launch failed */
  FLOWMOE_ERR_NCCL = 3,        /* an NCCL call failed or the communicator reported an async error */
  FLOWMOE_ERR_OOM = 4,         /* device allocation of a ctx workspace failed */
  FLOWMOE_ERR_UNSUPPORTED = 5, /* valid but not implemented shape (e.g. d_h not in {16,32,64,128}) */
  FLOWMOE_ERR_STATE = 6        /* call out of order (e.g. waiting on an unknown ticket) */
} flowmoe_status;

typedef enum { FLOWMOE_F32 = 0, FLOWMOE_BF16 = 1 } flowmoe_dtype;

/* How flowmoe_block_bwd writes weight gradients: ACCUMULATE adds into the
 * buffers (gradient accumulation across backward calls), OVERWRITE stores them
 * (the buffers need no zeroing; like zero_grad(set_to_none) + backward). */
typedef enum { FLOWMOE_GRAD_ACCUMULATE = 0, FLOWMOE_GRAD_OVERWRITE = 1 } flowmoe_grad_mode;

/* Scheduling policy — the paper's ablation (Table 6), all on
 * the same kernels and with identical results for the same effective R:
 *   FLOWMOE     AT, D, E, C split into R subtasks (Eqs.(3)-(6)) + chunked AR per block
 *   FLOWMOE_AR  MoE part split (experts + A2A), AT unsplit, chunked AR per block
 *   FLOWMOE_AT  AT and MoE part split, AR centralized after the backward pass
 *   PIPE_MOE    MoE part split only (Tutel-like), AT unsplit, AR centralized
 *   VANILLA_EP  no pipelining (R treated as 1), AR centralized */
typedef enum {
  FLOWMOE_SCHED_FLOWMOE = 0, FLOWMOE_SCHED_FLOWMOE_AR = 1, FLOWMOE_SCHED_FLOWMOE_AT = 2,
  FLOWMOE_SCHED_PIPE_MOE = 3, FLOWMOE_SCHED_VANILLA_EP = 4
} flowmoe_schedule;

/* A2A implementation: NCCL grouped send/recv, or peer-memory kernels over NVLink
 * (buffers mapped with CUDA IPC at create / first use of a `saved` stash — the first
 * flowmoe_block_fwd of each stash must run outside CUDA-graph capture on every rank,
 * otherwise that stash falls back to NCCL). */
typedef enum { FLOWMOE_A2A_NCCL = 0, FLOWMOE_A2A_P2P = 1 } flowmoe_a2a_impl;

typedef struct {
  int64_t B;               /* tokens on this rank (paper B·N); B % seq_len == 0; (B/seq_len) % R == 0 */
  int32_t seq_len;         /* N, tokens per sequence (attention span) */
  int32_t M;               /* model dim; M % n_heads == 0; d_h = M/n_heads in {16,32,64,128} */
  int32_t n_heads;         /* h (not in the paper; reading Q13) */
  int32_t E;               /* experts per block, E in {2,4,8,16,32,64}; E % world_size == 0 */
  int32_t top_k;           /* k, 1 <= k <= min(E, 8) */
  int32_t d_ffn;           /* expert hidden size (paper H), multiple of 8 */
  int32_t R;               /* pipelining degree, >= 1 */
  float capacity_factor;   /* f >= 0; 0 => dropless (C = B/R); else C = ceil(f·k·(B/R)/E) */
  int32_t causal;          /* 0/1: causal attention mask */
  int32_t residual;        /* 0/1: I' = ctx·Wo + x and y = MoE(I') + I' */
  int32_t dtype;           /* flowmoe_dtype */
  int32_t world_size;      /* P */
  int32_t rank;            /* p; experts [p·E/P, (p+1)·E/P) are local (reading Q12) */
  int32_t grad_mode;       /* flowmoe_grad_mode */
  int32_t compute_streams; /* 0/1: the compute tasks of all chunks run in Eq.(3)/(5) order on ONE
                              stream (the paper's single compute resource); n > 1: chunk r's
                              compute tasks run in that order on stream r % min(n, R), so chunks
                              whose kernels do not fill the 148 SMs co-run (same results) */
  int32_t schedule;        /* a flowmoe_schedule value; default FLOWMOE */
  int32_t a2a_impl;        /* a flowmoe_a2a_impl value: NCCL send/recv groups (default) or
                              stores from this library's kernels into CUDA-IPC-mapped peer
                              buffers on NVLink (world_size <= 8; results identical) */
} flowmoe_config;

/* Weights of one block (dtype of the config).  Replicated: wqkv [M][3M] (columns
 * q|k|v), wo [M][M], wg [M][E].  Local experts only: w1 [E/P][M][F],
 * b1 [E/P][F], w2 [E/P][F][M], b2 [E/P][M]. */
typedef struct {
  const void *wqkv, *wo, *wg, *w1, *b1, *w2, *b2;
} flowmoe_params;

/* Gradients, fp32, accumulated (+=) or overwritten per config.grad_mode.
 * grad_flat = [dWqkv (M×3M) | dWo (M×M) | dWg (M×E)], 4M²+M·E floats,
 * all-reduced (sum over ranks) by the AR that flowmoe_block_bwd submits (in
 * ACCUMULATE mode the previous contents are summed over ranks too).
 * dw1 [E/P][M][F], db1 [E/P][F], dw2 [E/P][F][M], db2 [E/P][M] are the local
 * experts' grads summed over all source ranks (no AR: experts are sharded). */
typedef struct {
  float *grad_flat, *dw1, *db1, *dw2, *db2;
} flowmoe_grads;

typedef struct flowmoe_ctx flowmoe_ctx;
typedef uint64_t flowmoe_ticket;

/* NCCL unique id for world_size > 1: call on rank 0, broadcast the 128 bytes to
 * the other ranks (e.g. over torch.distributed), pass to flowmoe_create. */
flowmoe_status flowmoe_get_unique_id(uint8_t id[128]);

/* Validate the config and create a ctx on `device` (streams, events, NCCL comms
 * for world_size > 1, backward workspaces).  `id` may be NULL when world_size == 1.
 * Collective over the world when world_size > 1. */
flowmoe_status flowmoe_create(const flowmoe_config* cfg, const uint8_t id[128], int device,
                              flowmoe_ctx** out);

/* Bytes of the per-block activation stash written by block_fwd, read by block_bwd. */
size_t flowmoe_saved_bytes(const flowmoe_ctx* ctx);

/* Number of floats of the flat replicated-grad buffer: 4M² + M·E. */
size_t flowmoe_grad_flat_count(const flowmoe_ctx* ctx);

/* Forward of one block: x [B][M] -> y [B][M] (dtype), saving activations in
 * `saved`.  Compute tasks AT_1..AT_R, E_1..E_R run in Eq.(3) order on the
 * compute stream; D_r, C_r (NCCL all-to-all, world_size > 1) in Eq.(4) order on
 * the high-priority comm stream.  Work is ordered after prior work on `stream`
 * and `stream` waits for its completion.  Collective when world_size > 1. */
flowmoe_status flowmoe_block_fwd(flowmoe_ctx* ctx, const flowmoe_params* params, const void* x,
                                 void* y, void* saved, cudaStream_t stream);

/* Backward of one block given dy [B][M]: dx [B][M] (nullable: skipped), grads
 * accumulated (+=).  `x` is the block's forward input [B][M] (the same pointer passed to
 * block_fwd; read by the deferred dWqkv = xᵀ·dQKV GEMM) — an extension of SURVEY §8(b)'s
 * signature, which would otherwise have to copy x into `saved` (B·M more bytes per block).  Compute order Eq.(5) (E_R..E_1, AT_R..AT_1), A2A order
 * Eq.(6).  The AR of grad_flat is auto-submitted in chunks of `chunk_bytes`
 * (S_p; positive multiple of 16; >= bytes => one chunk; last chunk is the
 * remainder) at priority 1 as soon as the grads are final
 * (P:1173), returned in *ar (nullable).  Call flowmoe_allreduce_wait before
 * reading grad_flat (Alg. 1 line 22). */
flowmoe_status flowmoe_block_bwd(flowmoe_ctx* ctx, const flowmoe_params* params, const void* x,
                                 const void* saved, const void* dy, void* dx,
                                 const flowmoe_grads* grads, size_t chunk_bytes,
                                 flowmoe_ticket* ar, cudaStream_t stream);

/* The L-block stack (Alg. 1 lines 6-21) in one call each way.  Same results
 * as L block_fwd / block_bwd calls; the lanes are forked once, so chunk r of block l+1
 * starts as soon as chunk r of block l is done (no block-boundary barrier).
 *   stack_fwd: block l maps ys[l-1] (x0 for l = 0) -> ys[l], stash saved[l].
 *   stack_bwd: blocks L-1..0; block l gets dy (l = L-1) or dxs[l+1], writes dxs[l]
 *              (dxs[0] nullable), grads[l], and returns its AR ticket in tickets[l]
 *              (nullable).  params/grads/ys/saved/dxs/tickets are arrays of length L. */
flowmoe_status flowmoe_stack_fwd(flowmoe_ctx* ctx, int L, const flowmoe_params* params, const void* x0,
                                 void* const* ys, void* const* saved, cudaStream_t stream);
flowmoe_status flowmoe_stack_bwd(flowmoe_ctx* ctx, int L, const flowmoe_params* params, const void* x0,
                                 void* const* ys, void* const* saved, const void* dy, void* const* dxs,
                                 const flowmoe_grads* grads, size_t chunk_bytes, flowmoe_ticket* tickets,
                                 cudaStream_t stream);

/* Optimizer (reading Q17: the paper updates each block's experts as soon as their
 * gradients are final — at E_1^l of the backward, P:1173 — and the replicated MHA/gate
 * weights after their all-reduce, but names no optimizer).  kind FLOWMOE_OPT_SGD:
 * d = g + wd·w, b = beta1·b + d (b = d at step 1), w -= lr·b (beta1 = momentum; beta2,
 * eps unused).  FLOWMOE_OPT_ADAMW: m = b1·m + (1-b1)·g, v = b2·v + (1-b2)·g²,
 * w = w·(1 - lr·wd) - lr·(m/(1-b1^t)) / (sqrt(v/(1-b2^t)) + eps). */
typedef enum { FLOWMOE_OPT_SGD = 0, FLOWMOE_OPT_ADAMW = 1 } flowmoe_opt_kind;
typedef struct {
  int32_t kind;  /* flowmoe_opt_kind */
  float lr, beta1, beta2, eps, weight_decay;
} flowmoe_optimizer;

/* One step over n elements on `stream`: fp32 master weights (updated in place), state1
 * (SGD momentum buffer / AdamW m) and state2 (AdamW v; NULL for SGD), fp32 gradient; if
 * `weight` is non-NULL the updated value is also written there in the config dtype (the
 * compute copy the block reads).  step >= 1 counts this tensor's updates.  Invalid
 * arguments return FLOWMOE_ERR_INVALID before anything is enqueued. */
flowmoe_status flowmoe_optimizer_step(flowmoe_ctx* ctx, const flowmoe_optimizer* opt, int64_t step, float* master,
                                      float* state1, float* state2, const float* grad, void* weight, size_t n,
                                      cudaStream_t stream);

/* ---- Model edges around the block stack ----
 * Token embedding, forward: x[t][:] = table[ids[t]][:] for t < T; table [V][M] and x
 * [T][M] in the config dtype, ids [T] int32 on the device; an id outside [0, V) gives a
 * zero row (ids are not validated on the host).  Backward: dtable[v][:] += Σ_{t: ids[t]=v}
 * dx[t][:] into an fp32 [V][M] gradient (ACCUMULATED, like flowmoe_grads), deterministic
 * (tokens added in t order, one writer per element).  M is the config's model dim; M·size
 * of the dtype must be a multiple of 16 bytes.  Errors: FLOWMOE_ERR_INVALID (NULL pointer,
 * T < 0, V < 1) before anything is enqueued. */
flowmoe_status flowmoe_embed_fwd(flowmoe_ctx* ctx, const void* table, int64_t V, const int32_t* ids, int64_t T,
                                 void* x, cudaStream_t stream);
flowmoe_status flowmoe_embed_bwd(flowmoe_ctx* ctx, const int32_t* ids, int64_t T, const void* dx, int64_t V,
                                 float* dtable, cudaStream_t stream);

/* Softmax cross-entropy over fp32 logits [T][V] with int32 labels [T] (label < 0 or >= V:
 * row ignored).  losses [T] fp32 (caller scratch) receives lse_t - l_t[y_t]; loss [1] fp32
 * (nullable) = scale · Σ_t losses[t]; dlogits [T][V] in the config dtype (nullable) =
 * scale · (softmax(l_t) - onehot(y_t)).  The chunked loss of Eqs.(19)-(23) is the sum of
 * per-chunk calls with scale = 1/T_total (reading Q18).  Deterministic (fixed-order
 * reductions).  Errors: FLOWMOE_ERR_INVALID (NULL logits/labels/losses, T < 0, V < 1). */
flowmoe_status flowmoe_xent(flowmoe_ctx* ctx, const float* logits, const int32_t* labels, int64_t T, int64_t V,
                            float scale, float* losses, float* loss, void* dlogits, cudaStream_t stream);

/* LM head (the projection between the last block and flowmoe_xent), tcgen05 GEMMs:
 * forward logits[T][V] (fp32) = h[T][M] · W[V][M]ᵀ; backward dh[T][M] = dlogits[T][V] · W
 * (config dtype, overwritten; nullable) and dW[V][M] += dlogitsᵀ · h (fp32, ACCUMULATED;
 * nullable).  h, W and dlogits in the config dtype, row-major, M = the config's model dim;
 * V must be a positive multiple of 8 (16-byte TMA strides).  Errors: FLOWMOE_ERR_INVALID
 * before anything is enqueued. */
flowmoe_status flowmoe_lm_head_fwd(flowmoe_ctx* ctx, const void* h, const void* w, int64_t T, int64_t V,
                                   float* logits, cudaStream_t stream);
flowmoe_status flowmoe_lm_head_bwd(flowmoe_ctx* ctx, const void* h, const void* w, const void* dlogits, int64_t T,
                                   int64_t V, void* dh, float* dw, cudaStream_t stream);

/* Per-tensor optimizer storage of the local experts, index 0..3 = w1, b1, w2, b2 (shapes of
 * flowmoe_params); weight[i] is the compute copy (the flowmoe_params pointer). */
typedef struct {
  float* master[4];
  float* state1[4];
  float* state2[4];
  void* weight[4];
} flowmoe_expert_opt;

/* Expert update of the block whose flowmoe_block_bwd / flowmoe_stack_bwd was enqueued last
 * with these grads: enqueued on the ctx's weight-gradient stream right behind that
 * block's expert wgrads, so it overlaps the rest of the backward and the all-reduces.
 * *done (nullable) receives a ticket: flowmoe_allreduce_wait(ctx, *done, s) makes stream s
 * wait for the update (before the next forward reads the weights). */
flowmoe_status flowmoe_expert_update(flowmoe_ctx* ctx, const flowmoe_optimizer* opt, int64_t step,
                                     const flowmoe_expert_opt* st, const flowmoe_grads* grads, flowmoe_ticket* done);

/* Chunked in-place sum all-reduce of buf[count] fp32 over the world on the
 * low-priority AR stream (Alg. 2 PARTITION + ARQueue).  Starts after `ready`
 * (nullable: after work already enqueued on the ctx compute stream).
 * priority >= 1 (lower = sooner; 0 is reserved for A2A).  world_size == 1: no-op. */
flowmoe_status flowmoe_allreduce_submit(flowmoe_ctx* ctx, float* buf, size_t count,
                                        size_t chunk_bytes, int priority, cudaEvent_t ready,
                                        flowmoe_ticket* out);

/* Make `stream` wait for every chunk of the ticket's all-reduce; polls NCCL async errors.
 * FLOWMOE_ERR_STATE for an unknown / expired ticket. */
flowmoe_status flowmoe_allreduce_wait(flowmoe_ctx* ctx, flowmoe_ticket ticket, cudaStream_t stream);

/* Peer-memory A2A (a2a_impl = FLOWMOE_A2A_P2P, world_size > 1): map a `saved` stash into
 * every peer (CUDA IPC).  Collective: every rank registers its stashes in the same order,
 * outside CUDA-graph capture, before the first flowmoe_block_fwd / stack_fwd that uses them;
 * the exchange is all-or-nothing (either every rank maps every peer or every rank gets
 * FLOWMOE_ERR_CUDA and the stash uses the NCCL path on all ranks).  A registered stash must
 * stay allocated until flowmoe_unregister_saved (or destroy): the peers keep writing into it.
 * Registering the same pointer again is a no-op; world_size == 1 or NCCL A2A: no-op.
 * A stash never registered is registered on first use (same rules; during capture it uses
 * NCCL).  unregister: local; synchronises the device, then closes this rank's mappings of
 * the peers' stashes (call it on every rank before freeing the stash anywhere). */
flowmoe_status flowmoe_register_saved(flowmoe_ctx* ctx, const void* saved);
flowmoe_status flowmoe_unregister_saved(flowmoe_ctx* ctx, const void* saved);

/* Health of the asynchronous exchange machinery, for callers that replay CUDA graphs (where
 * no host-side check runs): FLOWMOE_ERR_STATE / FLOWMOE_ERR_CUDA if a peer-memory A2A wait
 * timed out (~10-20 s without a peer's arrival; the waiting kernel then traps, faulting the
 * context, so consumers never read stale buffers), FLOWMOE_ERR_NCCL on an asynchronous NCCL
 * error.  Host-synchronous (reads one word from the device). */
flowmoe_status flowmoe_check_health(flowmoe_ctx* ctx);

/* Test hook: force the top-k indices ([B][k] int32 device array, distinct
 * experts per row) instead of selecting them; gate weights are still computed
 * from the logits at those indices.  NULL restores normal routing. */
flowmoe_status flowmoe_set_forced_routing(flowmoe_ctx* ctx, const int32_t* idx);

const char* flowmoe_status_string(flowmoe_status s);
const char* flowmoe_last_error(void); /* thread-local message of the last failing call */

/* Synchronises the ctx streams, destroys NCCL comms, frees workspaces. */
void flowmoe_destroy(flowmoe_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* FLOWMOE_H */
