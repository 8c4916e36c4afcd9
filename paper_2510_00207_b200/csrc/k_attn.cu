// K6 attention (S2 AT-attn, B5 attention backward) — flash-style, fp32 math.
// Per sequence s and head h: ctx = softmax(Q K^T / sqrt(d_h) [+causal]) V,
// saving lse = m + log(l) per row (P:75 MHA; reading Q7: no biases, 1/sqrt(d_h)).
// Backward (FlashAttention-2 order): D_i = rowsum(dO ⊙ O); P = exp(S - lse);
// dV = P^T dO; dP = dO V^T; dS = P ⊙ (dP - D); dK = dS^T Q / sqrt(d);
// dQ = dS K / sqrt(d).  dK/dV and dQ are computed by separate kernels so no
// atomics are needed (deterministic).  SIMT for round 1: attention is <= ~2%
// of block FLOPs at C3/C4; tcgen05 attention is NEXT.
#include "common.cuh"
#include "kernels.h"

namespace fm {

constexpr int AB = 64;  // rows per tile (queries or keys)

// row-major padded smem tile [AB][dh+1] (odd stride: conflict-free on both
// "one row per lane" and "one column per lane" access patterns)
template <typename T>
__device__ void load_tile(float* dst, const T* src, int64_t ld, int row0, int nrows, int dh) {
  const int vec = 16 / sizeof(T);
  const int per_row = dh / vec;
  for (int e = threadIdx.x; e < AB * per_row; e += blockDim.x) {
    int r = e / per_row, c = (e % per_row) * vec;
    float v[8];
    if (row0 + r < nrows) load16<T>(src + (int64_t)(row0 + r) * ld + c, v);
    else
#pragma unroll
      for (int i = 0; i < 8; ++i) v[i] = 0.f;
#pragma unroll
    for (int i = 0; i < vec; ++i) dst[r * (dh + 1) + c + i] = v[i];
  }
}

// Row ranges as in k_attn_tc.cu: own rows (queries for fwd / dQ, keys for dK/dV) are the
// positions [p0, p0 + np) of each of the n_seq sequences (N rows apart); whole sequences
// have p0 = 0, np = N; a token chunk is a slice of one sequence (causal).
// grid (ceil(np/AB), H, n_seq); 256 threads; thread (ty,tx): rows ty+16a (a<4),
// key cols tx+16b (b<4), output cols tx+16c (c<dh/16).
template <typename T, int DH>
__global__ void __launch_bounds__(256) attn_fwd_kernel(const T* qkv, T* ctx, float* lse, int N, int p0,
                                                       int np, int M, int H, int causal, float scale) {
  FM_PDL_ENTRY();
  extern __shared__ float sm[];
  float* Qs = sm;
  float* Ks = Qs + AB * (DH + 1);
  float* Vs = Ks + AB * (DH + 1);
  float* Ps = Vs + AB * (DH + 1);  // [AB][AB+1]
  const int qb = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t ld = 3 * (int64_t)M;
  const T* base = qkv + (int64_t)s * N * ld;
  const int pe = p0 + np;  // rows at or past pe are not read (not yet computed in a token chunk)
  load_tile<T>(Qs, base + h * DH, ld, p0 + qb * AB, pe, DH);
  constexpr int NC = DH / 16;
  float o[4][NC] = {};
  float mrow[4], lrow[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) { mrow[a] = -INFINITY; lrow[a] = 0.f; }
  const int nkb = causal ? (min(pe, p0 + (qb + 1) * AB) + AB - 1) / AB : (N + AB - 1) / AB;
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    load_tile<T>(Ks, base + M + h * DH, ld, kb * AB, pe, DH);
    load_tile<T>(Vs, base + 2 * M + h * DH, ld, kb * AB, pe, DH);
    __syncthreads();
    float sc[4][4] = {};
    for (int d = 0; d < DH; ++d) {
      float q[4], k[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) q[a] = Qs[(ty + 16 * a) * (DH + 1) + d];
#pragma unroll
      for (int b = 0; b < 4; ++b) k[b] = Ks[(tx + 16 * b) * (DH + 1) + d];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) sc[a][b] = fmaf(q[a], k[b], sc[a][b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = p0 + qb * AB + ty + 16 * a;
      float mx = -INFINITY;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = kb * AB + tx + 16 * b;
        bool valid = j < N && (!causal || j <= i);
        sc[a][b] = valid ? sc[a][b] * scale : -INFINITY;
        mx = fmaxf(mx, sc[a][b]);
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, off));
      const float mnew = fmaxf(mrow[a], mx);
      const float corr = (mrow[a] == -INFINITY) ? 0.f : expf(mrow[a] - mnew);
      float rs = 0.f;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        float p = (sc[a][b] == -INFINITY) ? 0.f : expf(sc[a][b] - mnew);
        Ps[(ty + 16 * a) * (AB + 1) + tx + 16 * b] = p;
        rs += p;
      }
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) rs += __shfl_xor_sync(0xffffffffu, rs, off);
      lrow[a] = lrow[a] * corr + rs;
      mrow[a] = mnew;
#pragma unroll
      for (int c = 0; c < NC; ++c) o[a][c] *= corr;
    }
    __syncthreads();
    for (int j = 0; j < AB; ++j) {
      float v[NC], p[4];
#pragma unroll
      for (int c = 0; c < NC; ++c) v[c] = Vs[j * (DH + 1) + tx + 16 * c];
#pragma unroll
      for (int a = 0; a < 4; ++a) p[a] = Ps[(ty + 16 * a) * (AB + 1) + j];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < NC; ++c) o[a][c] = fmaf(p[a], v[c], o[a][c]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = p0 + qb * AB + ty + 16 * a;
    if (i >= pe) continue;
    const float inv = 1.f / lrow[a];
    T* dst = ctx + ((int64_t)s * N + i) * M + h * DH;
#pragma unroll
    for (int c = 0; c < NC; ++c) dst[tx + 16 * c] = from_f<T>(o[a][c] * inv);
    if (tx == 0) lse[((int64_t)s * N + i) * H + h] = mrow[a] + logf(lrow[a]);
  }
}

// D[t][h] = sum_d dO[t][h*dh+d] * O[t][h*dh+d]
template <typename T>
__global__ void attn_bwd_pre_kernel(const T* ctx, const T* dctx, float* D, int T_, int M, int H) {
  FM_PDL_ENTRY();
  const int64_t id = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (int64_t)T_ * H) return;
  const int t = id / H, h = id % H, dh = M / H;
  const T* o = ctx + (int64_t)t * M + h * dh;
  const T* d = dctx + (int64_t)t * M + h * dh;
  float acc = 0.f;
  for (int c = 0; c < dh; ++c) acc = fmaf(to_f<T>(o[c]), to_f<T>(d[c]), acc);
  D[id] = acc;
}

// dK, dV for one own key block; grid (ceil(np/AB), H, n_seq); queries up to N.
// thread: keys ty+16a (a<4) x queries tx+16b (b<4); dK/dV rows ty+16a x cols tx+16c.
template <typename T, int DH>
__global__ void __launch_bounds__(256) attn_bwd_dkdv_kernel(const T* qkv, const T* dctx,
                                                            const float* lse, const float* D,
                                                            T* dqkv, int N, int p0, int np, int M, int H,
                                                            int causal, float scale) {
  FM_PDL_ENTRY();
  extern __shared__ float sm[];
  float* Ks = sm;
  float* Vs = Ks + AB * (DH + 1);
  float* Qs = Vs + AB * (DH + 1);
  float* dOs = Qs + AB * (DH + 1);
  float* Ps = dOs + AB * (DH + 1);   // [AB keys][AB+1]
  float* dSs = Ps + AB * (AB + 1);   // [AB keys][AB+1]
  float* Ls = dSs + AB * (AB + 1);   // lse of query rows
  float* Ds = Ls + AB;
  const int kb = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t ld = 3 * (int64_t)M;
  const T* base = qkv + (int64_t)s * N * ld;
  const T* dob = dctx + (int64_t)s * N * M;
  const int pe = p0 + np, k0 = p0 + kb * AB;
  load_tile<T>(Ks, base + M + h * DH, ld, k0, pe, DH);
  load_tile<T>(Vs, base + 2 * M + h * DH, ld, k0, pe, DH);
  constexpr int NC = DH / 16;
  float dk[4][NC] = {}, dv[4][NC] = {};
  const int nqb = (N + AB - 1) / AB;
  for (int qb = causal ? k0 / AB : 0; qb < nqb; ++qb) {
    __syncthreads();
    load_tile<T>(Qs, base + h * DH, ld, qb * AB, N, DH);
    load_tile<T>(dOs, dob + h * DH, M, qb * AB, N, DH);
    for (int r = tid; r < AB; r += blockDim.x) {
      int i = qb * AB + r;
      Ls[r] = i < N ? lse[((int64_t)s * N + i) * H + h] : 0.f;
      Ds[r] = i < N ? D[((int64_t)s * N + i) * H + h] : 0.f;
    }
    __syncthreads();
    float sc[4][4] = {}, dp[4][4] = {};
    for (int d = 0; d < DH; ++d) {
      float k[4], v[4], q[4], g[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) { k[a] = Ks[(ty + 16 * a) * (DH + 1) + d]; v[a] = Vs[(ty + 16 * a) * (DH + 1) + d]; }
#pragma unroll
      for (int b = 0; b < 4; ++b) { q[b] = Qs[(tx + 16 * b) * (DH + 1) + d]; g[b] = dOs[(tx + 16 * b) * (DH + 1) + d]; }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) { sc[a][b] = fmaf(k[a], q[b], sc[a][b]); dp[a][b] = fmaf(v[a], g[b], dp[a][b]); }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int j = k0 + ty + 16 * a;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int il = tx + 16 * b, i = qb * AB + il;
        bool valid = i < N && j < pe && (!causal || j <= i);
        float p = valid ? expf(sc[a][b] * scale - Ls[il]) : 0.f;
        Ps[(ty + 16 * a) * (AB + 1) + il] = p;
        dSs[(ty + 16 * a) * (AB + 1) + il] = valid ? p * (dp[a][b] - Ds[il]) : 0.f;
      }
    }
    __syncthreads();
    for (int i = 0; i < AB; ++i) {
      float q[NC], g[NC], p[4], ds[4];
#pragma unroll
      for (int c = 0; c < NC; ++c) { q[c] = Qs[i * (DH + 1) + tx + 16 * c]; g[c] = dOs[i * (DH + 1) + tx + 16 * c]; }
#pragma unroll
      for (int a = 0; a < 4; ++a) { p[a] = Ps[(ty + 16 * a) * (AB + 1) + i]; ds[a] = dSs[(ty + 16 * a) * (AB + 1) + i]; }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < NC; ++c) { dv[a][c] = fmaf(p[a], g[c], dv[a][c]); dk[a][c] = fmaf(ds[a], q[c], dk[a][c]); }
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int j = k0 + ty + 16 * a;
    if (j >= pe) continue;
    T* row = dqkv + ((int64_t)s * N + j) * ld;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      row[M + h * DH + tx + 16 * c] = from_f<T>(dk[a][c] * scale);
      row[2 * M + h * DH + tx + 16 * c] = from_f<T>(dv[a][c]);
    }
  }
}

// dQ for one own query block; grid (ceil(np/AB), H, n_seq).
// thread: queries ty+16a x keys tx+16b; dQ rows ty+16a x cols tx+16c.
template <typename T, int DH>
__global__ void __launch_bounds__(256) attn_bwd_dq_kernel(const T* qkv, const T* dctx,
                                                          const float* lse, const float* D,
                                                          T* dqkv, int N, int p0, int np, int M, int H,
                                                          int causal, float scale) {
  FM_PDL_ENTRY();
  extern __shared__ float sm[];
  float* Qs = sm;
  float* dOs = Qs + AB * (DH + 1);
  float* Ks = dOs + AB * (DH + 1);
  float* Vs = Ks + AB * (DH + 1);
  float* dSs = Vs + AB * (DH + 1);  // [AB queries][AB+1]
  const int qb = blockIdx.x, h = blockIdx.y, s = blockIdx.z;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const int64_t ld = 3 * (int64_t)M;
  const T* base = qkv + (int64_t)s * N * ld;
  const int pe = p0 + np, q0 = p0 + qb * AB;
  load_tile<T>(Qs, base + h * DH, ld, q0, pe, DH);
  load_tile<T>(dOs, dctx + (int64_t)s * N * M + h * DH, M, q0, pe, DH);
  float L[4], Dv[4];
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    int i = q0 + ty + 16 * a;
    L[a] = i < pe ? lse[((int64_t)s * N + i) * H + h] : 0.f;
    Dv[a] = i < pe ? D[((int64_t)s * N + i) * H + h] : 0.f;
  }
  constexpr int NC = DH / 16;
  float dq[4][NC] = {};
  const int nkb = causal ? (min(pe, q0 + AB) + AB - 1) / AB : (N + AB - 1) / AB;
  for (int kb = 0; kb < nkb; ++kb) {
    __syncthreads();
    load_tile<T>(Ks, base + M + h * DH, ld, kb * AB, causal ? pe : N, DH);
    load_tile<T>(Vs, base + 2 * M + h * DH, ld, kb * AB, causal ? pe : N, DH);
    __syncthreads();
    float sc[4][4] = {}, dp[4][4] = {};
    for (int d = 0; d < DH; ++d) {
      float q[4], g[4], k[4], v[4];
#pragma unroll
      for (int a = 0; a < 4; ++a) { q[a] = Qs[(ty + 16 * a) * (DH + 1) + d]; g[a] = dOs[(ty + 16 * a) * (DH + 1) + d]; }
#pragma unroll
      for (int b = 0; b < 4; ++b) { k[b] = Ks[(tx + 16 * b) * (DH + 1) + d]; v[b] = Vs[(tx + 16 * b) * (DH + 1) + d]; }
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) { sc[a][b] = fmaf(q[a], k[b], sc[a][b]); dp[a][b] = fmaf(g[a], v[b], dp[a][b]); }
    }
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int i = q0 + ty + 16 * a;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int j = kb * AB + tx + 16 * b;
        bool valid = i < pe && j < N && (!causal || j <= i);
        float p = valid ? expf(sc[a][b] * scale - L[a]) : 0.f;
        dSs[(ty + 16 * a) * (AB + 1) + tx + 16 * b] = valid ? p * (dp[a][b] - Dv[a]) : 0.f;
      }
    }
    __syncthreads();
    for (int j = 0; j < AB; ++j) {
      float k[NC], ds[4];
#pragma unroll
      for (int c = 0; c < NC; ++c) k[c] = Ks[j * (DH + 1) + tx + 16 * c];
#pragma unroll
      for (int a = 0; a < 4; ++a) ds[a] = dSs[(ty + 16 * a) * (AB + 1) + j];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < NC; ++c) dq[a][c] = fmaf(ds[a], k[c], dq[a][c]);
    }
  }
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int i = q0 + ty + 16 * a;
    if (i >= pe) continue;
    T* row = dqkv + ((int64_t)s * N + i) * ld + h * DH;
#pragma unroll
    for (int c = 0; c < NC; ++c) row[tx + 16 * c] = from_f<T>(dq[a][c] * scale);
  }
}

template <typename T, int DH>
static int attn_fwd_t(const void* qkv, void* ctx, float* lse, int nseq, int N, int p0, int np, int M, int H,
                      int causal, cudaStream_t s) {
  size_t smem = (3 * AB * (DH + 1) + AB * (AB + 1)) * sizeof(float);
  auto k = attn_fwd_kernel<T, DH>;
  static bool once = (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), true);
  (void)once;
  dim3 grid((np + AB - 1) / AB, H, nseq);
  launch_k(k, grid, 256, smem, s, (const T*)qkv, (T*)ctx, lse, N, p0, np, M, H, causal, 1.0f / sqrtf((float)DH));
  return (int)cudaGetLastError();
}

template <typename T, int DH>
static int attn_bwd_t(const void* qkv, const void* ctx, const float* lse, const void* dctx,
                      void* dqkv, float* D, int nseq, int N, int p0, int np, int M, int H, int causal,
                      cudaStream_t s) {
  const float scale = 1.0f / sqrtf((float)DH);
  // D of the own rows (contiguous: either whole sequences or one slice of one sequence);
  // a token chunk's dK/dV reads the D rows of the later chunks, computed before it
  const int nrow = (nseq - 1) * N + np;
  launch_k(attn_bwd_pre_kernel<T>, (nrow * H + 255) / 256, 256, 0, s, (const T*)ctx + (int64_t)p0 * M,
           (const T*)dctx + (int64_t)p0 * M, D + (int64_t)p0 * H, nrow, M, H);
  dim3 grid((np + AB - 1) / AB, H, nseq);
  size_t smem1 = (4 * AB * (DH + 1) + 2 * AB * (AB + 1) + 2 * AB) * sizeof(float);
  auto k1 = attn_bwd_dkdv_kernel<T, DH>;
  static bool once1 = (cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem1), true);
  (void)once1;
  launch_k(k1, grid, 256, smem1, s, (const T*)qkv, (const T*)dctx, lse, D, (T*)dqkv, N, p0, np, M, H, causal,
           scale);
  size_t smem2 = (4 * AB * (DH + 1) + AB * (AB + 1)) * sizeof(float);
  auto k2 = attn_bwd_dq_kernel<T, DH>;
  static bool once2 = (cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2), true);
  (void)once2;
  launch_k(k2, grid, 256, smem2, s, (const T*)qkv, (const T*)dctx, lse, D, (T*)dqkv, N, p0, np, M, H, causal,
           scale);
  return (int)cudaGetLastError();
}

#define FM_DH_SWITCH(dh, F, ...)                 \
  switch (dh) {                                  \
    case 16: return F<16>(__VA_ARGS__);          \
    case 32: return F<32>(__VA_ARGS__);          \
    case 64: return F<64>(__VA_ARGS__);          \
    case 128: return F<128>(__VA_ARGS__);        \
    default: return (int)cudaErrorInvalidValue;  \
  }

template <int DH> static int fwd_f32(const void* a, void* b, float* c, int d, int e, int p0, int np, int f, int g, int h, cudaStream_t s) { return attn_fwd_t<float, DH>(a, b, c, d, e, p0, np, f, g, h, s); }
template <int DH> static int fwd_bf16(const void* a, void* b, float* c, int d, int e, int p0, int np, int f, int g, int h, cudaStream_t s) { return attn_fwd_t<bf16, DH>(a, b, c, d, e, p0, np, f, g, h, s); }
template <int DH> static int bwd_f32(const void* a, const void* b, const float* c, const void* d, void* e, float* f, int g, int h, int p0, int np, int i, int j, int k, cudaStream_t s) { return attn_bwd_t<float, DH>(a, b, c, d, e, f, g, h, p0, np, i, j, k, s); }
template <int DH> static int bwd_bf16(const void* a, const void* b, const float* c, const void* d, void* e, float* f, int g, int h, int p0, int np, int i, int j, int k, cudaStream_t s) { return attn_bwd_t<bf16, DH>(a, b, c, d, e, f, g, h, p0, np, i, j, k, s); }

int attn_fwd(int dtype, const void* qkv, void* ctx, float* lse, int nseq, int N, int p0, int np, int M, int H,
             int causal, cudaStream_t s) {
  if (attn_tc_supported(dtype, M, H)) return attn_fwd_tc(qkv, ctx, lse, nseq, N, p0, np, M, H, causal, s);
  const int dh = M / H;
  if (dtype == DT_F32) { FM_DH_SWITCH(dh, fwd_f32, qkv, ctx, lse, nseq, N, p0, np, M, H, causal, s) }
  FM_DH_SWITCH(dh, fwd_bf16, qkv, ctx, lse, nseq, N, p0, np, M, H, causal, s)
}

int attn_bwd(int dtype, const void* qkv, const void* ctx, const float* lse, const void* dctx,
             void* dqkv, float* D, int nseq, int N, int p0, int np, int M, int H, int causal, cudaStream_t s) {
  if (attn_tc_supported(dtype, M, H))
    return attn_bwd_tc(qkv, ctx, lse, dctx, dqkv, D, nseq, N, p0, np, M, H, causal, s);
  const int dh = M / H;
  if (dtype == DT_F32) { FM_DH_SWITCH(dh, bwd_f32, qkv, ctx, lse, dctx, dqkv, D, nseq, N, p0, np, M, H, causal, s) }
  FM_DH_SWITCH(dh, bwd_bf16, qkv, ctx, lse, dctx, dqkv, D, nseq, N, p0, np, M, H, causal, s)
}

}  // namespace fm
