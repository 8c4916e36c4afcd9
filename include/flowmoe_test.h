/* flowmoe_test.h — test, inspection and benchmark hooks of libflowmoe.so.
 *
 * NOT part of the product ABI (include/flowmoe.h): these calls exist so the parity tests
 * (tests/) and bench.py can look inside the block (routing decisions in the `saved` stash),
 * drive single kernels, time kernels, and simulate several ranks on one GPU.  Same
 * conventions as flowmoe.h (return codes, thread-local message, nothing throws).  Knobs and
 * profiles are per ctx: they are installed into the kernel modules at the start of each
 * enqueueing call of that ctx (not thread-safe across ctxs driven from several threads).
 */
#ifndef FLOWMOE_TEST_H
#define FLOWMOE_TEST_H

#include "flowmoe.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Byte offsets inside `saved` of the fp32 gate logits [B][E], indices [B][k]
 * int32, gate weights [B][k] fp32, positions [B][k] int32 (-1 = dropped) and
 * per-chunk counts [R][E] int32 (test inspection of routing). */
flowmoe_status flowmoe_saved_routing_offsets(const flowmoe_ctx* ctx, size_t* logits, size_t* idx,
                                             size_t* w, size_t* pos, size_t* counts);

/* Per-ctx test/benchmark knobs: key 1 = force the SIMT GEMM for bf16 (debug), key 2 =
 * swap MN-major descriptor strides (debug), key 3 = force the SIMT attention
 * kernels for bf16 (debug / A-B comparison), key 4 = programmatic dependent
 * launch on (1, default) / off (0), key 5 = force the GEMM tile width (64/128/256;
 * 0 = automatic), key 6 = peer-memory A2A of chunk r on chunk r's compute lane (1,
 * default) / on the A2A stream (0), key 7 = GEMM CTA grouping (0 automatic, 1 one CTA
 * per 128-row tile, 2 CTA pairs on 256-row tiles with cta_group::2 UMMAs), key 8 = GEMM
 * stream-K (0 automatic, 1 never, 2 wherever the GEMM has enough k-blocks: every SM / pair
 * gets the same share of the flattened (tile, k-block) space, cut tiles are summed in a
 * fixed order), key 9 = SMs the backward GEMMs leave free for the all-reduce at P > 1 (the
 * persistent GEMM grids shrink to 148 - value SMs; default the AR communicator's CTA cap,
 * 32, on a multi-process ctx, 0 in the simulated world), key 10 = SMs every GEMM leaves to
 * the other lanes' kernels (0 default).  Returns
 * FLOWMOE_ERR_INVALID on an unknown key. */
flowmoe_status flowmoe_debug_set(flowmoe_ctx* ctx, int key, int value);

/* Test hook: one GEMM through the block's GEMM kernels (tcgen05 for BF16,
 * fp32 SIMT for F32), with ctx's knobs and profile (ctx nullable: library defaults).
 * C(m,n) = epi(sum_k A(m,k) B(k,n)) per batch b, with
 * A(m,k) = A[b*sA + m*lda + k] (a_mmajor=0) or A[b*sA + k*lda + m] (a_mmajor=1),
 * B(k,n) = B[b*sB + k*ldb + n] (b_kmajor=0) or B[b*sB + n*ldb + k] (b_kmajor=1).
 * epi: 0 store (+bias[n] +resid), 1 bias+GELU (aux = pre-activation),
 * 2 times GELU'(aux), 3 fp32 accumulate C += acc, 4 fp32 store, 5 bias+GELU with
 * aux = GELU'(pre-activation), 6 times aux.  bias/resid/aux nullable;
 * resid and aux share C's ld/stride, bias has stride N per batch. */
flowmoe_status flowmoe_test_gemm(flowmoe_ctx* ctx, int dtype, int M, int N, int K, int batch, const void* A,
                                 int64_t lda, int64_t sA, int a_mmajor, const void* B, int64_t ldb,
                                 int64_t sB, int b_kmajor, void* C, int64_t ldc, int64_t sC, int epi,
                                 const void* bias, const void* resid, void* aux, cudaStream_t stream);

/* Per-kernel device timing of one ctx.  Between begin and end, every kernel / NCCL
 * call the library enqueues for that ctx outside CUDA-graph capture is
 * bracketed by timing events on its own stream.  end synchronises the device
 * and writes one entry per kernel kind that ran: launches, summed device ms,
 * summed algorithmic FLOPs and HBM (or bus) bytes.  While profiling, the
 * compute lanes are collapsed onto one stream so every duration is the
 * kernel's own.  Returns the number of entries written, or -1 on error. */
typedef struct {
  const char* name;   /* static string owned by the library */
  int64_t launches;
  double ms, flops, bytes;
} flowmoe_prof_entry;
flowmoe_status flowmoe_profile_begin(flowmoe_ctx* ctx);
int flowmoe_profile_end(flowmoe_ctx* ctx, flowmoe_prof_entry* out, int max_entries);

/* Task log of one ctx (eager enqueues only; SURVEY §8(c.3) schedule properties): between
 * begin and end every task the ctx enqueues is bracketed by timing events on its own
 * stream.  kind: 0 AT_r, 1 D_r, 2 E_r, 3 C_r, 4 merge_r (forward); 5 C_r^bwd pack,
 * 6 C_r^bwd exchange, 7 E_r^bwd, 8 D_r^bwd exchange, 9 expert wgrads (chunk -1),
 * 10 AT_r^bwd, 11 MHA/gate wgrads (chunk -1), 12 an all-reduce chunk (chunk = its index in
 * the S_p partition).  block = the call's index within the log window per direction
 * (dir 0 forward, 1 backward: stack_bwd's first block is the stack's last); chunk r = -1
 * for the unsplit-AT policies' single AT task; stream = cudaStreamGetId of the stream;
 * t0/t1 = ms since the window began.  end synchronises the device and returns the number
 * of records written (-1 on error).  The timing events break programmatic-launch overlap
 * between tasks, so logged runs are slower than unlogged ones (orders and dependencies are
 * unchanged). */
typedef struct {
  int32_t kind, block, chunk, dir;
  uint64_t stream;
  double t0_ms, t1_ms;
} flowmoe_task_rec;
flowmoe_status flowmoe_tasklog_begin(flowmoe_ctx* ctx);
int flowmoe_tasklog_end(flowmoe_ctx* ctx, flowmoe_task_rec* out, int max_entries);

/* Number of kernels this library has launched in the calling process (bench accounting). */
uint64_t flowmoe_kernel_launches(void);

/* Bus-bandwidth probe: `iters` back-to-back exchanges of chunk r of a registered `saved`
 * stash (kind 0: dispatch D_r owner -> expert side, 1: combine C_r back), through the ctx's
 * A2A implementation (NCCL send/recv groups or the peer-memory kernel), ordered after the
 * work on `stream` and waited for by it.  Collective; world_size > 1 (NCCL world) only. */
flowmoe_status flowmoe_test_exchange(flowmoe_ctx* ctx, void* saved, int kind, int r, int iters, cudaStream_t stream);

/* The peer-memory A2A arrival counters of this rank: out[(kind·R + r)·P + src] = how many
 * times source rank `src` has delivered exchange `kind` (0 D_r, 1 C_r, 2 C_r^bwd, 3 D_r^bwd)
 * of chunk r into this rank (monotonic).  n >= 4·R·world_size.  Synchronises the device.
 * FLOWMOE_ERR_STATE without a peer-memory A2A. */
flowmoe_status flowmoe_test_arrivals(const flowmoe_ctx* ctx, unsigned int* out, size_t n);

/* In-process simulated world for one-GPU tests of the exchange rows (S6/S8/B1/B3 peer-
 * memory A2A kernels and arrival counters, B6 S_p chunking of the all-reduce): P ctxs
 * (2 <= P <= 8; out[P]) of world_size P, ranks 0..P-1, on ONE device, peers' buffers mapped
 * as plain device pointers (a2a_impl forced to P2P; no NCCL).  The all-reduce of a
 * submission runs once every rank made its matching submission: the P ranks' buffers are
 * summed chunk by chunk (the same S_p partition as the NCCL path) in rank order on a group
 * stream and the sum is written back to every rank; flowmoe_allreduce_wait on a ticket whose
 * peers have not submitted yet returns FLOWMOE_ERR_STATE.  Each rank must register its
 * `saved` stashes (flowmoe_register_saved) before the first forward.  Drive every rank from
 * its own host thread: no kernel waits for another launch on the device (nothing guarantees
 * that separate launches on one GPU run at the same time); instead each exchange records an
 * event after this rank's send kernel, the member threads meet at a host barrier (120 s
 * timeout: FLOWMOE_ERR_STATE), and every rank's stream waits for its peers' send events.
 * Not capturable into a CUDA graph.  Call allreduce_wait after every rank's backward.  Schedules FLOWMOE and FLOWMOE_AR only (the centralized-AR
 * policies flush inside allreduce_wait, before the other ranks could submit).  Destroy every
 * member with flowmoe_destroy; each drains the device first. */
flowmoe_status flowmoe_create_local_group(const flowmoe_config* cfg, int P, int device, flowmoe_ctx** out);

#ifdef __cplusplus
}
#endif
#endif /* FLOWMOE_TEST_H */
