// Internal launcher interface between the FlowMoE scheduler (flowmoe.cu) and
// the sm_100a kernels.  Not part of the public C ABI (include/flowmoe.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace fm {

enum DType { DT_F32 = 0, DT_BF16 = 1 };

// ---------------------------------------------------------------- GEMM
// C(m,n) = epilogue( alpha * sum_k A(m,k) B(k,n) ), batched over `batch`.
//   A(m,k) = A[b*sA + m*lda + k]   (a_mmajor = 0, "K-major")
//          = A[b*sA + k*lda + m]   (a_mmajor = 1, "M-major": A stored transposed)
//   B(k,n) = B[b*sB + k*ldb + n]   (b_kmajor = 0: weights W[in][out], "N-major")
//          = B[b*sB + n*ldb + k]   (b_kmajor = 1: B = W^T, "K-major")
// Epilogues (all math in fp32):
//   EPI_STORE     C = alpha*acc (+ bias[n]) (+ resid(m,n))          -> storage dtype
//   EPI_BIAS_GELU aux = Z = acc + bias[n];  C = GELU(Z)             -> storage dtype
//   EPI_DGELU     C = acc * GELU'(aux(m,n))                        -> storage dtype
//   EPI_ACC_F32   Cf32(m,n) += alpha*acc                            -> fp32 (grads, accumulate)
//   EPI_STORE_F32 Cf32(m,n)  = alpha*acc                            -> fp32 (grads, overwrite)
//   EPI_BIAS_GELU_G  z = bf16(acc + bias[n]);  C = GELU(z), aux = GELU'(z)   -> storage dtype
//   EPI_MUL_AUX      C = acc * aux(m,n)                              -> storage dtype
// The expert FFN uses the last two: the forward saves GELU'(Z) instead of Z, so the
// backward's dZ = dH ⊙ GELU'(Z) epilogue is one multiply instead of erf + exp per element.
enum GemmEpi {
  EPI_STORE = 0, EPI_BIAS_GELU = 1, EPI_DGELU = 2, EPI_ACC_F32 = 3, EPI_STORE_F32 = 4,
  EPI_BIAS_GELU_G = 5, EPI_MUL_AUX = 6
};

struct GemmArgs {
  int M = 0, N = 0, K = 0, batch = 1;
  const void* A = nullptr; int64_t lda = 0, sA = 0; int a_mmajor = 0;
  const void* B = nullptr; int64_t ldb = 0, sB = 0; int b_kmajor = 0;
  void* C = nullptr; int64_t ldc = 0, sC = 0;
  const void* bias = nullptr; int64_t sBias = 0;
  const void* resid = nullptr; int64_t ldr = 0, sR = 0;
  void* aux = nullptr; int64_t ldaux = 0, sAux = 0;
  int epi = EPI_STORE;
  float alpha = 1.0f;
  // optional stream-K scratch (k_gemm_tc.cu): one fp32 128 x BN partial tile per CTA of the
  // grid, and one "partials written" counter per cut tile and CTA of the pair (zeroed once;
  // every use leaves them zero).  Without it the GEMM never splits a tile.
  float* splitk_ws = nullptr;
  size_t splitk_ws_floats = 0;
  unsigned int* splitk_tick = nullptr;
  size_t splitk_ticks = 0;
  int max_sms = 0;  // > 0: persistent grid on at most this many SMs (the rest left to a collective)
};

// Dispatches to the tcgen05 kernel for bf16 and the fp32 SIMT kernel (K10) for f32.
int gemm(const GemmArgs& g, int dtype, cudaStream_t s);
int gemm_simt(const GemmArgs& g, int dtype, cudaStream_t s);
int gemm_tc(const GemmArgs& g, cudaStream_t s);  // bf16 only, tcgen05/TMEM/TMA
int gemm_tc_init();                               // resolves cuTensorMapEncodeTiled
void gemm_tc_set_debug(int flags);
void gemm_tc_force_bn(int bn);
void gemm_tc_force_cg(int cg);
void gemm_tc_force_streamk(int mode);  // 0 automatic, 1 never, 2 wherever the scratch allows  // 0 automatic, 1 single-CTA tiles, 2 CTA pairs (cta_group::2)

// ---------------------------------------------------------------- attention
// qkv [nseq·N][3M] (sequences of N rows; head h at columns h*dh of each of Q|K|V),
// ctx [..][M], lse [..][H] fp32; all pointers at the first sequence's row 0.
// Own rows = positions [p0, p0+np) of every sequence: whole sequences p0 = 0, np = N;
// a token chunk (chunked prefill, causal only, nseq = 1) attends to keys [0, p0+np) and
// reads no row at or past p0+np in the forward.  The backward's dK/dV of the own keys
// takes every query up to N (their dctx rows must be final).
int attn_fwd(int dtype, const void* qkv, void* ctx, float* lse, int nseq, int N, int p0, int np, int M,
             int H, int causal, cudaStream_t s);
// dctx [..][M] -> own rows of dqkv [..][3M]; Dbuf [..][H] fp32 scratch.
int attn_bwd(int dtype, const void* qkv, const void* ctx, const float* lse, const void* dctx,
             void* dqkv, float* Dbuf, int nseq, int N, int p0, int np, int M, int H, int causal,
             cudaStream_t s);

// tcgen05 flash attention (bf16, d_h in {64,128}); attn_fwd/attn_bwd dispatch to these.
bool attn_tc_supported(int dtype, int M, int H);
int attn_tc_debug_off();
int attn_fwd_tc(const void* qkv, void* ctx, float* lse, int nseq, int N, int p0, int np, int M, int H,
                int causal, cudaStream_t s);
int attn_bwd_tc(const void* qkv, const void* ctx, const float* lse, const void* dctx, void* dqkv,
                float* D, int nseq, int N, int p0, int np, int M, int H, int causal, cudaStream_t s);

// ---------------------------------------------------------------- routing / data movement
// K1: logits = a·Wg (fp32), top-k (ties -> lower index), gate weights.
int gate_topk(int dtype, const void* a, const void* wg, const int32_t* forced, float* logits,
              int32_t* idx, float* w, int T, int M, int E, int k, cudaStream_t s);
// K1+K2 fused: the last CTA of the gate kernel runs the routing scan of the chunk.
// done: one zero-initialised counter per concurrently running chunk (reset in-kernel).
int gate_route(int dtype, const void* a, const void* wg, const int32_t* forced, float* logits,
               int32_t* idx, float* w, int32_t* pos, int32_t* counts, int32_t* src, unsigned int* done,
               int T, int M, int E, int k, int C, cudaStream_t s);
// K2: deterministic slot-major positions; counts[E]; src[E][C] = t*k+j or -1; pos[T][k] (-1 dropped)
int route_scan(const int32_t* idx, int32_t* pos, int32_t* counts, int32_t* src, int T, int E,
               int k, int C, cudaStream_t s);
// Owner-side expert buffers are [E][R][C][M] (expert-major, chunk-minor); a chunk's
// view starts at r*C rows and consecutive experts are ldE = R*C rows apart.
// K3: send[e*ldE + c] = a[src/k] or zeros, for (e, c) in [E) x [C).
int permute_pack(int dtype, const void* a, const int32_t* src, void* send, int E, int C, int ldE,
                 int M, int k, cudaStream_t s);
// K7: out[t] = sum_j w_tj * y[idx][pos] (+ a[t] if resid)
int unpermute_combine(int dtype, const void* y, const int32_t* idx, const int32_t* pos,
                      const float* w, const void* resid, void* out, int T, int M, int k, int ldE,
                      cudaStream_t s);
// K8: dy[e][pos] = w * dO[t]; dw[t][j] = <dO[t], y[e][pos]>; padding rows zeroed.
int combine_bwd_pack(int dtype, const void* dout, const void* y, const int32_t* idx,
                     const int32_t* pos, const float* w, const int32_t* src, void* dy, float* dw,
                     int T, int M, int k, int E, int C, int ldE, cudaStream_t s);
// K9: dA[t] = sum_j dx[e][pos] + dlogits·Wg^T (+ dO[t] if resid); dlogits [T][E] fp32 out.
int gather_gate_bwd(int dtype, const void* dx, const int32_t* idx, const int32_t* pos,
                    const float* w, const float* dw, const float* logits, const void* wg,
                    const void* dout_resid, void* dA, float* dlogits, int T, int M, int E, int k,
                    int ldE, cudaStream_t s);
// dWg[M][E] (+)= A^T · dlogits (deterministic split-T partials); part: scratch [nsplit][M][E]
int gate_wgrad(int dtype, const void* a, const float* dlogits, float* dwg, float* part, int T,
               int M, int E, int accumulate, cudaStream_t s);
size_t gate_wgrad_scratch_floats(int T, int M, int E);
// out[b][n] (+)= sum_r X[b][r][n]   (bias gradients)
int colsum_acc(int dtype, const void* x, float* out, int batch, int rows, int N, int accumulate,
               cudaStream_t s);

// Optimizer step (k_optim.cu): kind 0 SGD-momentum (s1 = momentum buffer, b1 = momentum),
// 1 AdamW (s1 = m, s2 = v); fp32 master w; out = compute copy in `dtype` (nullable).
int optim_step(int dtype, int kind, float lr, float b1, float b2, float eps, float wd, int64_t step, float* w,
               float* s1, float* s2, const float* g, void* out, int64_t n, cudaStream_t s);

// Model edges (k_model.cu): token embedding and softmax cross-entropy.
int embed_fwd(int dtype, const void* table, const int32_t* ids, void* x, int64_t T_, int64_t V, int M,
              cudaStream_t s);
int embed_bwd(int dtype, const int32_t* ids, const void* dx, float* dtable, int64_t T_, int64_t V, int M,
              cudaStream_t s);
int xent(int dtype, const float* logits, const int32_t* labels, int64_t T_, int64_t V, float scale, float* losses,
         float* loss, void* dlogits, cudaStream_t s);

// A2A over NVLink peer memory (k_p2p.cu): send (copy + publish) and/or wait for (kind, r).
int a2a_p2p(const void* src, void* const* dst, unsigned int* const* peer_flags, unsigned int* piece_cnt,
            unsigned int* my_flags, unsigned int* seen, unsigned int* err, int kind, int r, int R, int P,
            int El, int me, int to_experts, int64_t blk_bytes, cudaStream_t send_stream,
            cudaStream_t wait_stream, bool do_send, bool do_wait, unsigned int* grid_cnt = nullptr);

// Simulated world all-reduce (flowmoe_create_local_group): bufs[q][off, off+n) of the P
// ranks summed in rank order and written back to all of them; 16-byte aligned chunk starts.
int local_allreduce(float* const* bufs, int P, int64_t off, int64_t n, cudaStream_t s);

}  // namespace fm
