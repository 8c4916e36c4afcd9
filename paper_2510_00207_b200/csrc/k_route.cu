// Gating, routing and token movement kernels of the FlowMoE block.
//   K1 gate_topk        (S4: logits = I'·Wg, softmax, top-k)
//   K2 route_scan       (S5: capacity positions C = ceil(f·k·B·N/E))
//   K3 permute_pack     (S5: rows -> A2A send buffer G(I') ∈ R^{E×C×M})
//   K7 unpermute_combine(S9: out[t] = Σ_j w_tj·Y[e_tj][pos_tj] (+I'))
//   K8 combine_bwd_pack (B1: dY = w·dO, dw = <dO, Y>)
//   K9 gather_gate_bwd  (B4: dI' = Σ dX + dlogits·Wgᵀ (+dO))
//   gate_wgrad          (B4: dWg += I'ᵀ·dlogits, deterministic split-T)
//   colsum_acc          (B2: db1, db2)
// All HBM-bound: one warp per token row with 16-byte vector accesses.
// Readings: Q3 slot-major-then-token positions, Q4 top-k on fp32
// logits with ties -> lower index, Q5 renormalised top-k weights (k>=2) or raw
// softmax prob (k=1), Q6 no gate bias.
#include "common.cuh"
#include "kernels.h"

namespace fm {

// E contiguous storage elements -> fp32 (16-byte vector loads when the row allows)
template <typename T, int E>
FM_DEV void load_row(const T* p, float* out) {
  constexpr int V = 16 / sizeof(T);
  if constexpr (E % V == 0) {
#pragma unroll
    for (int i = 0; i < E; i += V) load16<T>(p + i, out + i);
  } else {
#pragma unroll
    for (int i = 0; i < E; ++i) out[i] = to_f<T>(p[i]);
  }
}

__device__ void route_scan_body(const int32_t* idx, int32_t* pos, int32_t* counts, int32_t* src, int T_,
                                int E, int k, int C, int* hist, int* warp_tot);

// ------------------------------------------------------------------ K1
// One warp per token.  Lane l owns row elements [8l + 256i, 8l + 256i + 8) (bf16)
// or [4l + 128i, ...) (f32) and keeps E partial dot products; xor-reduce gives
// every lane all E logits, then top-k by repeated argmax (strictly greater ->
// lower index wins ties).
// With `done` != nullptr the kernel also runs K2: the CTA that finishes last (atomic
// ticket on done[0], reset afterwards) performs the deterministic routing scan of the
// whole chunk, saving a launch.
template <typename T, int E>
__global__ void __launch_bounds__(256) gate_topk_kernel(const T* a, const T* wg,
                                                        const int32_t* forced, float* logits,
                                                        int32_t* idx, float* w, int T_, int M,
                                                        int k, int32_t* pos, int32_t* counts,
                                                        int32_t* src, int C, unsigned int* done) {
  FM_PDL_ENTRY();
  extern __shared__ int hist[];  // [E][blockDim.x] for the fused scan
  __shared__ int warp_tot[32];
  __shared__ unsigned int ticket;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp < T_) {
  constexpr int V = 16 / sizeof(T);
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  const T* row = a + (int64_t)warp * M;
  for (int m0 = lane * V; m0 < M; m0 += 32 * V) {
    float x[8];
    load16<T>(row + m0, x);
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float wr[E];
      load_row<T, E>(wg + (int64_t)(m0 + i) * E, wr);
#pragma unroll
      for (int e = 0; e < E; ++e) acc[e] = fmaf(x[i], wr[e], acc[e]);
    }
  }
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = warp_sum(acc[e]);
  if (lane < E) {
    float mine = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) if (e == lane) mine = acc[e];
    logits[(int64_t)warp * E + lane] = mine;
  }
  if (lane == 0) {
  // top-k selection on logits
  uint64_t taken = 0;
  int sel[8];
  for (int j = 0; j < k; ++j) {
    int best = -1;
    float bv = 0.f;
    if (forced) {
      best = forced[(int64_t)warp * k + j];
    } else {
#pragma unroll
      for (int e = 0; e < E; ++e)
        if (!((taken >> e) & 1ull) && (best < 0 || acc[e] > bv)) { best = e; bv = acc[e]; }
    }
    taken |= 1ull << best;
    sel[j] = best;
    idx[(int64_t)warp * k + j] = best;
  }
  float lsel[8];
  for (int j = 0; j < k; ++j) {
    float v = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) if (e == sel[j]) v = acc[e];
    lsel[j] = v;
  }
  if (k == 1) {
    // w0 = p_{e0} = 1 / Σ_e exp(l_e - l_e0)
    float den = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) den += expf(acc[e] - lsel[0]);
    w[warp] = 1.f / den;
  } else {
    float mx = lsel[0];
    for (int j = 1; j < k; ++j) mx = fmaxf(mx, lsel[j]);
    float den = 0.f, ex[8];
    for (int j = 0; j < k; ++j) { ex[j] = expf(lsel[j] - mx); den += ex[j]; }
    for (int j = 0; j < k; ++j) w[(int64_t)warp * k + j] = ex[j] / den;
  }
  }  // lane 0
  }  // warp < T_
  if (done == nullptr) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) ticket = atomicAdd(done, 1u);
  __syncthreads();
  if (ticket != gridDim.x - 1) return;
  __threadfence();  // every CTA's idx is visible
  route_scan_body(idx, pos, counts, src, T_, E, k, C, hist, warp_tot);
  if (threadIdx.x == 0) *done = 0u;  // ready for the next use (stream-ordered)
}

#define FM_E_SWITCH(E_, F, ...)                                 \
  switch (E_) {                                                 \
    case 2: F<2>(__VA_ARGS__); break;                           \
    case 4: F<4>(__VA_ARGS__); break;                           \
    case 8: F<8>(__VA_ARGS__); break;                           \
    case 16: F<16>(__VA_ARGS__); break;                         \
    case 32: F<32>(__VA_ARGS__); break;                         \
    case 64: F<64>(__VA_ARGS__); break;                         \
    default: return (int)cudaErrorInvalidValue;                 \
  }

template <int E>
static void gate_topk_launch(int dtype, const void* a, const void* wg, const int32_t* forced,
                             float* logits, int32_t* idx, float* w, int T_, int M, int k,
                             int32_t* pos, int32_t* counts, int32_t* src, int C, unsigned int* done,
                             cudaStream_t s) {
  dim3 grid((T_ * 32 + 255) / 256);
  const size_t smem = done ? (size_t)E * 256 * sizeof(int) : 0;
  if (dtype == DT_F32) {
    static bool once = (cudaFuncSetAttribute(gate_topk_kernel<float, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             E * 256 * (int)sizeof(int)), true);
    (void)once;
    launch_k(gate_topk_kernel<float, E>, grid, 256, smem, s, (const float*)a, (const float*)wg, forced,
             logits, idx, w, T_, M, k, pos, counts, src, C, done);
  } else {
    static bool once = (cudaFuncSetAttribute(gate_topk_kernel<bf16, E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             E * 256 * (int)sizeof(int)), true);
    (void)once;
    launch_k(gate_topk_kernel<bf16, E>, grid, 256, smem, s, (const bf16*)a, (const bf16*)wg, forced,
             logits, idx, w, T_, M, k, pos, counts, src, C, done);
  }
}

int gate_topk(int dtype, const void* a, const void* wg, const int32_t* forced, float* logits,
              int32_t* idx, float* w, int T_, int M, int E, int k, cudaStream_t s) {
  if (T_ <= 0) return 0;
  FM_E_SWITCH(E, gate_topk_launch, dtype, a, wg, forced, logits, idx, w, T_, M, k, nullptr, nullptr,
              nullptr, 0, nullptr, s)
  return (int)cudaGetLastError();
}

int gate_route(int dtype, const void* a, const void* wg, const int32_t* forced, float* logits,
               int32_t* idx, float* w, int32_t* pos, int32_t* counts, int32_t* src, unsigned int* done,
               int T_, int M, int E, int k, int C, cudaStream_t s) {
  if (T_ <= 0) return 0;
  FM_E_SWITCH(E, gate_topk_launch, dtype, a, wg, forced, logits, idx, w, T_, M, k, pos, counts, src,
              C, done, s)
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K2
// One CTA per chunk.  Slots in slot-major order s = j*T + t are split into
// contiguous per-thread segments; pass 1 counts per expert, a block-wide
// exclusive scan per expert gives every thread its starting position, pass 2
// re-walks the segment assigning pos = base[e]++.  Deterministic: pos equals
// the number of earlier slots (in slot-major order) routed to the same expert.
constexpr int RS_THREADS = 512;

__device__ int block_excl_scan(int v, int* warp_tot) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    int t = lane < (int)(blockDim.x >> 5) ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  int res = x - v + (wid > 0 ? warp_tot[wid - 1] : 0);
  __syncthreads();
  return res;
}

// Block-wide deterministic routing scan (one CTA, any block size <= 1024): hist is
// [E][blockDim.x] ints of dynamic shared memory.
__device__ void route_scan_body(const int32_t* idx, int32_t* pos, int32_t* counts, int32_t* src, int T_,
                                int E, int k, int C, int* hist, int* warp_tot) {
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = T_ * k;
  const int seg = (n + nt - 1) / nt;
  const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
  for (int e = 0; e < E; ++e) hist[e * nt + tid] = 0;
  for (int i = tid; i < E * C; i += nt) src[i] = -1;
  for (int s = s0; s < s1; ++s) {
    const int j = s / T_, t = s % T_;
    hist[idx[(int64_t)t * k + j] * nt + tid] += 1;
  }
  __syncthreads();
  for (int e = 0; e < E; ++e) {
    int v = hist[e * nt + tid];
    int ex = block_excl_scan(v, warp_tot);
    hist[e * nt + tid] = ex;
    if (tid == nt - 1) counts[e] = ex + v;
  }
  __syncthreads();
  for (int s = s0; s < s1; ++s) {
    const int j = s / T_, t = s % T_;
    const int e = idx[(int64_t)t * k + j];
    const int p = hist[e * nt + tid]++;
    const bool kept = p < C;
    pos[(int64_t)t * k + j] = kept ? p : -1;
    if (kept) src[e * C + p] = t * k + j;
  }
}

__global__ void __launch_bounds__(RS_THREADS) route_scan_kernel(const int32_t* idx, int32_t* pos,
                                                                int32_t* counts, int32_t* src,
                                                                int T_, int E, int k, int C) {
  FM_PDL_ENTRY();
  extern __shared__ int hist[];  // [E][RS_THREADS]
  __shared__ int warp_tot[32];
  route_scan_body(idx, pos, counts, src, T_, E, k, C, hist, warp_tot);
}

int route_scan(const int32_t* idx, int32_t* pos, int32_t* counts, int32_t* src, int T_, int E,
               int k, int C, cudaStream_t s) {
  size_t smem = (size_t)E * RS_THREADS * sizeof(int);
  static bool once = (cudaFuncSetAttribute(route_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           64 * RS_THREADS * (int)sizeof(int)), true);
  (void)once;
  launch_k(route_scan_kernel, 1, RS_THREADS, smem, s, idx, pos, counts, src, T_, E, k, C);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K3
template <typename T>
__global__ void __launch_bounds__(256) permute_pack_kernel(const T* a, const int32_t* src,
                                                           T* send, int rows, int C, int ldE,
                                                           int M, int k) {
  FM_PDL_ENTRY();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int sl = src[warp];
  constexpr int V = 16 / sizeof(T);
  const int64_t drow = (int64_t)(warp / C) * ldE + warp % C;
  uint4* dst = reinterpret_cast<uint4*>(send + drow * M);
  const int nv = M / V;
  if (sl < 0) {
    for (int i = lane; i < nv; i += 32) dst[i] = make_uint4(0, 0, 0, 0);
  } else {
    const uint4* srow = reinterpret_cast<const uint4*>(a + (int64_t)(sl / k) * M);
    for (int i = lane; i < nv; i += 32) dst[i] = __ldg(srow + i);
  }
}

int permute_pack(int dtype, const void* a, const int32_t* src, void* send, int E, int C, int ldE,
                 int M, int k, cudaStream_t s) {
  const int rows = E * C;
  if (rows <= 0) return 0;
  dim3 grid((rows * 32 + 255) / 256);
  if (dtype == DT_F32)
    launch_k(permute_pack_kernel<float>, grid, 256, 0, s, (const float*)a, src, (float*)send, rows, C, ldE, M, k);
  else
    launch_k(permute_pack_kernel<bf16>, grid, 256, 0, s, (const bf16*)a, src, (bf16*)send, rows, C, ldE, M, k);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K7
template <typename T>
__global__ void __launch_bounds__(256) unpermute_combine_kernel(const T* y, const int32_t* idx,
                                                                const int32_t* pos, const float* w,
                                                                const T* resid, T* out, int T_,
                                                                int M, int k, int ldE) {
  FM_PDL_ENTRY();
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T_) return;
  constexpr int V = 16 / sizeof(T);
  const T* rows[8];
  float ws[8];
  int nk = 0;
  for (int j = 0; j < k; ++j) {
    int p = pos[(int64_t)t * k + j];
    if (p >= 0) {
      rows[nk] = y + ((int64_t)idx[(int64_t)t * k + j] * ldE + p) * M;
      ws[nk] = w[(int64_t)t * k + j];
      ++nk;
    }
  }
  for (int m0 = lane * V; m0 < M; m0 += 32 * V) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < nk; ++j) {
      float v[8];
      load16<T>(rows[j] + m0, v);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = fmaf(ws[j], v[i], acc[i]);
    }
    if (resid) {
      float v[8];
      load16<T>(resid + (int64_t)t * M + m0, v);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += v[i];
    }
    store16<T>(out + (int64_t)t * M + m0, acc);
  }
}

int unpermute_combine(int dtype, const void* y, const int32_t* idx, const int32_t* pos,
                      const float* w, const void* resid, void* out, int T_, int M, int k, int ldE,
                      cudaStream_t s) {
  if (T_ <= 0) return 0;
  dim3 grid((T_ * 32 + 255) / 256);
  if (dtype == DT_F32)
    launch_k(unpermute_combine_kernel<float>, grid, 256, 0, s, (const float*)y, idx, pos, w,
                                                        (const float*)resid, (float*)out, T_, M, k, ldE);
  else
    launch_k(unpermute_combine_kernel<bf16>, grid, 256, 0, s, (const bf16*)y, idx, pos, w,
                                                       (const bf16*)resid, (bf16*)out, T_, M, k, ldE);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K8
// warps [0, T): token work; warps [T, T + E*C): zero the padding rows of dy.
template <typename T>
__global__ void __launch_bounds__(256) combine_bwd_pack_kernel(const T* dout, const T* y,
                                                               const int32_t* idx,
                                                               const int32_t* pos, const float* w,
                                                               const int32_t* src, T* dy,
                                                               float* dw, int T_, int M, int k,
                                                               int rows, int C, int ldE) {
  FM_PDL_ENTRY();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  constexpr int V = 16 / sizeof(T);
  if (warp >= T_) {
    const int r = warp - T_;
    if (r >= rows || src[r] >= 0) return;
    uint4* dst = reinterpret_cast<uint4*>(dy + ((int64_t)(r / C) * ldE + r % C) * M);
    for (int i = lane; i < M / V; i += 32) dst[i] = make_uint4(0, 0, 0, 0);
    return;
  }
  const int t = warp;
  const T* g = dout + (int64_t)t * M;
  for (int j = 0; j < k; ++j) {
    const int p = pos[(int64_t)t * k + j];
    if (p < 0) {  // dropped slot: contributes 0, so dw = 0
      if (lane == 0) dw[(int64_t)t * k + j] = 0.f;
      continue;
    }
    const int64_t row = (int64_t)idx[(int64_t)t * k + j] * ldE + p;
    const float wj = w[(int64_t)t * k + j];
    float dot = 0.f;
    for (int m0 = lane * V; m0 < M; m0 += 32 * V) {
      float gv[8], yv[8], o[8];
      load16<T>(g + m0, gv);
      load16<T>(y + row * M + m0, yv);
#pragma unroll
      for (int i = 0; i < V; ++i) { dot = fmaf(gv[i], yv[i], dot); o[i] = wj * gv[i]; }
      store16<T>(dy + row * M + m0, o);
    }
    dot = warp_sum(dot);
    if (lane == 0) dw[(int64_t)t * k + j] = dot;
  }
}

int combine_bwd_pack(int dtype, const void* dout, const void* y, const int32_t* idx,
                     const int32_t* pos, const float* w, const int32_t* src, void* dy, float* dw,
                     int T_, int M, int k, int E, int C, int ldE, cudaStream_t s) {
  const int rows = E * C;
  dim3 grid(((T_ + rows) * 32 + 255) / 256);
  if (dtype == DT_F32)
    launch_k(combine_bwd_pack_kernel<float>, grid, 256, 0, s, (const float*)dout, (const float*)y, idx,
                                                       pos, w, src, (float*)dy, dw, T_, M, k, rows, C, ldE);
  else
    launch_k(combine_bwd_pack_kernel<bf16>, grid, 256, 0, s, (const bf16*)dout, (const bf16*)y, idx,
                                                      pos, w, src, (bf16*)dy, dw, T_, M, k, rows, C, ldE);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K9
template <typename T, int E>
__global__ void __launch_bounds__(256) gather_gate_bwd_kernel(
    const T* dx, const int32_t* idx, const int32_t* pos, const float* w, const float* dw,
    const float* logits, const T* wg, const T* dres, T* dA, float* dlogits, int T_, int M, int k,
    int ldE) {
  FM_PDL_ENTRY();
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T_) return;
  constexpr int V = 16 / sizeof(T);
  // dlogits (reading Q5): k>=2: dl_{e_j} = w_j (dw_j - Σ w dw); k=1: dl = p ⊙ (g - <p,g>)
  float dl[E];
#pragma unroll
  for (int e = 0; e < E; ++e) dl[e] = 0.f;
  const float* lt = logits + (int64_t)t * E;
  if (k == 1) {
    const int e0 = idx[t];
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < E; ++e) mx = fmaxf(mx, lt[e]);
    float den = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) { dl[e] = expf(lt[e] - mx); den += dl[e]; }
    const float g0 = dw[t];
    float pe0 = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) { dl[e] /= den; if (e == e0) pe0 = dl[e]; }
    // <p, g> = p_e0 * g0
#pragma unroll
    for (int e = 0; e < E; ++e) dl[e] = dl[e] * ((e == e0 ? g0 : 0.f) - pe0 * g0);
  } else {
    float inner = 0.f;
    for (int j = 0; j < k; ++j) inner += w[(int64_t)t * k + j] * dw[(int64_t)t * k + j];
    for (int j = 0; j < k; ++j) {
      const int ej = idx[(int64_t)t * k + j];
      const float v = w[(int64_t)t * k + j] * (dw[(int64_t)t * k + j] - inner);
#pragma unroll
      for (int e = 0; e < E; ++e) if (e == ej) dl[e] += v;
    }
  }
  if (lane < E) {
    float mine = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) if (e == lane) mine = dl[e];
    dlogits[(int64_t)t * E + lane] = mine;
  }
  const T* rows[8];
  int nk = 0;
  for (int j = 0; j < k; ++j) {
    const int p = pos[(int64_t)t * k + j];
    if (p >= 0) rows[nk++] = dx + ((int64_t)idx[(int64_t)t * k + j] * ldE + p) * M;
  }
  for (int m0 = lane * V; m0 < M; m0 += 32 * V) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int j = 0; j < nk; ++j) {
      float v[8];
      load16<T>(rows[j] + m0, v);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += v[i];
    }
#pragma unroll
    for (int i = 0; i < V; ++i) {
      float wr[E];
      load_row<T, E>(wg + (int64_t)(m0 + i) * E, wr);
      float s = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) s = fmaf(dl[e], wr[e], s);
      acc[i] += s;
    }
    if (dres) {
      float v[8];
      load16<T>(dres + (int64_t)t * M + m0, v);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] += v[i];
    }
    store16<T>(dA + (int64_t)t * M + m0, acc);
  }
}

template <int E>
static void gather_gate_bwd_launch(int dtype, const void* dx, const int32_t* idx,
                                   const int32_t* pos, const float* w, const float* dw,
                                   const float* logits, const void* wg, const void* dres, void* dA,
                                   float* dlogits, int T_, int M, int k, int ldE, cudaStream_t s) {
  dim3 grid((T_ * 32 + 255) / 256);
  if (dtype == DT_F32)
    launch_k(gather_gate_bwd_kernel<float, E>, grid, 256, 0, s, 
        (const float*)dx, idx, pos, w, dw, logits, (const float*)wg, (const float*)dres,
        (float*)dA, dlogits, T_, M, k, ldE);
  else
    launch_k(gather_gate_bwd_kernel<bf16, E>, grid, 256, 0, s, 
        (const bf16*)dx, idx, pos, w, dw, logits, (const bf16*)wg, (const bf16*)dres, (bf16*)dA,
        dlogits, T_, M, k, ldE);
}

int gather_gate_bwd(int dtype, const void* dx, const int32_t* idx, const int32_t* pos,
                    const float* w, const float* dw, const float* logits, const void* wg,
                    const void* dres, void* dA, float* dlogits, int T_, int M, int E, int k, int ldE,
                    cudaStream_t s) {
  if (T_ <= 0) return 0;
  FM_E_SWITCH(E, gather_gate_bwd_launch, dtype, dx, idx, pos, w, dw, logits, wg, dres, dA,
              dlogits, T_, M, k, ldE, s)
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ dWg
// part[sp][m][e] = Σ_{t in split sp} A[t][m] dl[t][e]; then dwg[m][e] += Σ_sp part (in order).
constexpr int GW_SPLIT_T = 32;

template <typename T, int E>
__global__ void __launch_bounds__(128) gate_wgrad_part_kernel(const T* a, const float* dl,
                                                              float* part, int T_, int M) {
  FM_PDL_ENTRY();
  __shared__ float dls[GW_SPLIT_T][E];
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  const int t0 = blockIdx.y * GW_SPLIT_T;
  const int nt = min(GW_SPLIT_T, T_ - t0);
  for (int i = threadIdx.x; i < nt * E; i += blockDim.x) dls[i / E][i % E] = dl[(int64_t)t0 * E + i];
  __syncthreads();
  if (m >= M) return;
  float acc[E];
#pragma unroll
  for (int e = 0; e < E; ++e) acc[e] = 0.f;
  for (int t = 0; t < nt; ++t) {
    const float x = to_f<T>(a[(int64_t)(t0 + t) * M + m]);
#pragma unroll
    for (int e = 0; e < E; ++e) acc[e] = fmaf(x, dls[t][e], acc[e]);
  }
  float* dst = part + ((int64_t)blockIdx.y * M + m) * E;
#pragma unroll
  for (int e = 0; e < E; ++e) dst[e] = acc[e];
}

__global__ void gate_wgrad_reduce_kernel(const float* part, float* dwg, int nsplit, int n, int accumulate) {
  FM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  float s = 0.f;
  for (int p = 0; p < nsplit; ++p) s += part[(int64_t)p * n + i];
  dwg[i] = accumulate ? dwg[i] + s : s;
}

size_t gate_wgrad_scratch_floats(int T_, int M, int E) {
  return (size_t)((T_ + GW_SPLIT_T - 1) / GW_SPLIT_T) * M * E;
}

template <int E>
static void gate_wgrad_launch(int dtype, const void* a, const float* dl, float* part, int T_,
                              int M, cudaStream_t s) {
  dim3 grid((M + 127) / 128, (T_ + GW_SPLIT_T - 1) / GW_SPLIT_T);
  if (dtype == DT_F32)
    launch_k(gate_wgrad_part_kernel<float, E>, grid, 128, 0, s, (const float*)a, dl, part, T_, M);
  else
    launch_k(gate_wgrad_part_kernel<bf16, E>, grid, 128, 0, s, (const bf16*)a, dl, part, T_, M);
}

int gate_wgrad(int dtype, const void* a, const float* dlogits, float* dwg, float* part, int T_,
               int M, int E, int accumulate, cudaStream_t s) {
  if (T_ <= 0) return 0;
  FM_E_SWITCH(E, gate_wgrad_launch, dtype, a, dlogits, part, T_, M, s)
  const int nsplit = (T_ + GW_SPLIT_T - 1) / GW_SPLIT_T;
  launch_k(gate_wgrad_reduce_kernel, (M * E + 255) / 256, 256, 0, s, part, dwg, nsplit, M * E, accumulate);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ bias grads
// out[b][n] (+)= Σ_r x[b][r][n].  Block (32 columns x 8 row groups): thread (tx, ty)
// sums rows ty, ty+8, ...; the 8 partials are added in a fixed order (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) colsum_acc_kernel(const T* x, float* out, int rows, int N, int accumulate) {
  FM_PDL_ENTRY();
  __shared__ float part[8][33];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int n = blockIdx.x * 32 + tx, b = blockIdx.y;
  const T* xb = x + (int64_t)b * rows * N;
  float s = 0.f;
  if (n < N)
    for (int r = ty; r < rows; r += 8) s += to_f<T>(xb[(int64_t)r * N + n]);
  part[ty][tx] = s;
  __syncthreads();
  if (ty == 0 && n < N) {
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += part[i][tx];
    out[(int64_t)b * N + n] = accumulate ? out[(int64_t)b * N + n] + t : t;
  }
}

int colsum_acc(int dtype, const void* x, float* out, int batch, int rows, int N, int accumulate,
               cudaStream_t s) {
  dim3 grid((N + 31) / 32, batch);
  if (dtype == DT_F32) launch_k(colsum_acc_kernel<float>, grid, 256, 0, s, (const float*)x, out, rows, N, accumulate);
  else launch_k(colsum_acc_kernel<bf16>, grid, 256, 0, s, (const bf16*)x, out, rows, N, accumulate);
  return (int)cudaGetLastError();
}

}  // namespace fm
