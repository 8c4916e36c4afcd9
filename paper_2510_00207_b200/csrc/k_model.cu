// Model edges around the block stack: token embedding
// (forward gather, deterministic backward scatter-add) and the softmax cross-entropy
// with its gradient, scaled so that the per-chunk losses of Eqs.(19)-(23) add up to the
// mean over all tokens (scale = 1/T per chunk; reading Q18).  All HBM / latency bound:
// 16-byte vectors, one CTA per logits row, fixed-order reductions (deterministic).
#include "common.cuh"
#include "kernels.h"

namespace fm {

// x[t][:] = table[ids[t]][:]; a warp per token; ids outside [0, V) give a zero row
template <typename T>
__global__ void __launch_bounds__(256) embed_fwd_kernel(const T* __restrict__ table, const int32_t* __restrict__ ids,
                                                        T* __restrict__ x, int64_t T_, int64_t V, int M) {
  FM_PDL_ENTRY();
  const int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (t >= T_) return;
  const int nv = M * (int)sizeof(T) / 16;
  const int64_t id = ids[t];
  uint4* dst = reinterpret_cast<uint4*>(x + t * M);
  if (id < 0 || id >= V) {
    for (int i = lane; i < nv; i += 32) dst[i] = make_uint4(0, 0, 0, 0);
    return;
  }
  const uint4* src = reinterpret_cast<const uint4*>(table + id * M);
  for (int i = lane; i < nv; i += 32) dst[i] = __ldg(src + i);
}

// dtable[v] += Σ_{t : ids[t] = v} dx[t] (fp32), tokens added in t order.  CTA (vb, cb)
// owns vocabulary rows [vb·EB_ROWS, +EB_ROWS) and a column block; it walks the ids in
// tiles, compacts the tokens that hit its rows in t order (ballot + warp offsets), and
// each thread adds those rows into its own columns — every (v, column) has exactly one
// writer, so no atomics and a fixed summation order.
constexpr int EB_ROWS = 256, EB_TILE = 1024;

template <typename T>
__global__ void __launch_bounds__(256) embed_bwd_kernel(const int32_t* __restrict__ ids, const T* __restrict__ dx,
                                                        float* __restrict__ dtable, int64_t T_, int64_t V, int M) {
  __shared__ int s_hit[EB_TILE];
  __shared__ int s_wcnt[8];
  FM_PDL_ENTRY();
  constexpr int VE = 16 / sizeof(T);  // columns per 16-byte vector
  const int64_t v0 = (int64_t)blockIdx.x * EB_ROWS;
  const int c = ((int)blockIdx.y * (int)blockDim.x + (int)threadIdx.x) * VE;  // first column
  const bool col_ok = c < M;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t base = 0; base < T_; base += EB_TILE) {
    // ordered compaction of this tile's hits: 4 ids per thread, thread-major inside a warp
    int flags = 0;
    int64_t tt[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      tt[q] = base + (int64_t)warp * 128 + q * 32 + lane;
      const int64_t id = tt[q] < T_ ? ids[tt[q]] : -1;
      if (id >= v0 && id < v0 + EB_ROWS && id < V) flags |= 1 << q;
    }
    unsigned int bal[4];
    int wtot = 0;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      bal[q] = __ballot_sync(0xffffffffu, (flags >> q) & 1);
      wtot += __popc(bal[q]);
    }
    if (lane == 0) s_wcnt[warp] = wtot;
    __syncthreads();
    int off = 0, ntot = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < warp) off += s_wcnt[w];
      ntot += s_wcnt[w];
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {  // a warp's ids are ordered q-major (q·32 + lane)
      if ((flags >> q) & 1) s_hit[off + __popc(bal[q] & ((1u << lane) - 1u))] = (int)(tt[q] - base);
      off += __popc(bal[q]);
    }
    __syncthreads();
    if (col_ok)
      for (int h = 0; h < ntot; ++h) {
        const int64_t t = base + s_hit[h];
        const int64_t v = ids[t];
        float g[VE];
        load16<T>(dx + t * M + c, g);
        float* d = dtable + v * M + c;
#pragma unroll
        for (int i = 0; i < VE; ++i) d[i] += g[i];
      }
    __syncthreads();
  }
}

// Per row t with label y_t >= 0: lse_t = log Σ_v exp(l_tv); loss_t = lse_t - l_ty;
// dlogits_tv = scale·(exp(l_tv - lse_t) - [v = y_t]).  Rows with y_t < 0 are ignored
// (loss 0, zero gradient).  One CTA per row: strided max / sum-of-exp per thread, warp
// butterflies and a fixed-order cross-warp sum (deterministic).
template <typename T>
__global__ void __launch_bounds__(256) xent_row_kernel(const float* __restrict__ logits, const int32_t* __restrict__ labels,
                                                       float* __restrict__ losses, T* __restrict__ dlogits,
                                                       int64_t V, float scale) {
  __shared__ float s_red[8];
  FM_PDL_ENTRY();
  const int64_t t = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float* l = logits + t * V;
  const int y = labels[t];
  const bool valid = y >= 0 && y < V;
  float mx = -INFINITY;
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) mx = fmaxf(mx, l[v]);
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) s_red[warp] = mx;
  __syncthreads();
  mx = s_red[0];
  for (int w = 1; w < 8; ++w) mx = fmaxf(mx, s_red[w]);
  __syncthreads();
  float se = 0.f;
  for (int64_t v = threadIdx.x; v < V; v += blockDim.x) se += expf(l[v] - mx);
  se = warp_sum(se);
  if (lane == 0) s_red[warp] = se;
  __syncthreads();
  se = 0.f;
  for (int w = 0; w < 8; ++w) se += s_red[w];
  const float lse = mx + logf(se);
  if (threadIdx.x == 0) losses[t] = valid ? lse - l[y] : 0.f;
  if (dlogits) {
    T* d = dlogits + t * V;
    for (int64_t v = threadIdx.x; v < V; v += blockDim.x) {
      const float g = valid ? scale * (expf(l[v] - lse) - (v == y ? 1.f : 0.f)) : 0.f;
      d[v] = from_f<T>(g);
    }
  }
}

// loss = scale · Σ_t losses[t], one CTA, fixed order (thread-strided partials, then warps)
__global__ void __launch_bounds__(256) xent_sum_kernel(const float* __restrict__ losses, int64_t T_, float scale,
                                                       float* __restrict__ loss) {
  __shared__ float s_red[8];
  FM_PDL_ENTRY();
  float s = 0.f;
  for (int64_t t = threadIdx.x; t < T_; t += blockDim.x) s += losses[t];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    float a = 0.f;
    for (int w = 0; w < 8; ++w) a += s_red[w];
    *loss = scale * a;
  }
}

int embed_fwd(int dtype, const void* table, const int32_t* ids, void* x, int64_t T_, int64_t V, int M,
              cudaStream_t s) {
  if (T_ <= 0) return 0;
  const dim3 grid((unsigned)((T_ + 7) / 8));
  if (dtype == DT_F32)
    launch_k(embed_fwd_kernel<float>, grid, 256, 0, s, (const float*)table, ids, (float*)x, T_, V, M);
  else
    launch_k(embed_fwd_kernel<bf16>, grid, 256, 0, s, (const bf16*)table, ids, (bf16*)x, T_, V, M);
  return (int)cudaGetLastError();
}

int embed_bwd(int dtype, const int32_t* ids, const void* dx, float* dtable, int64_t T_, int64_t V, int M,
              cudaStream_t s) {
  if (T_ <= 0 || V <= 0) return 0;
  const int ve = dtype == DT_F32 ? 4 : 8;
  const dim3 grid((unsigned)((V + EB_ROWS - 1) / EB_ROWS), (unsigned)((M + 256 * ve - 1) / (256 * ve)));
  if (dtype == DT_F32)
    launch_k(embed_bwd_kernel<float>, grid, 256, 0, s, ids, (const float*)dx, dtable, T_, V, M);
  else
    launch_k(embed_bwd_kernel<bf16>, grid, 256, 0, s, ids, (const bf16*)dx, dtable, T_, V, M);
  return (int)cudaGetLastError();
}

int xent(int dtype, const float* logits, const int32_t* labels, int64_t T_, int64_t V, float scale, float* losses,
         float* loss, void* dlogits, cudaStream_t s) {
  if (T_ <= 0) {
    if (loss) cudaMemsetAsync(loss, 0, sizeof(float), s);
    return (int)cudaGetLastError();
  }
  if (dtype == DT_F32)
    launch_k(xent_row_kernel<float>, dim3((unsigned)T_), 256, 0, s, logits, labels, losses, (float*)dlogits, V, scale);
  else
    launch_k(xent_row_kernel<bf16>, dim3((unsigned)T_), 256, 0, s, logits, labels, losses, (bf16*)dlogits, V, scale);
  if (loss) launch_k(xent_sum_kernel, dim3(1), 256, 0, s, (const float*)losses, T_, scale, loss);
  return (int)cudaGetLastError();
}

}  // namespace fm
