// K10 gemm_simt_f32: true-fp32 FFMA GEMM (dense + batched) with the FlowMoE
// epilogues.  Used by the fp32 parity mode (paper: "All parameters and
// gradients ... 32-bit single precision"), where TF32 tensor cores
// (10-bit mantissa) would miss the 1e-4 bound (SURVEY.md §7 hard part 7).
// The bf16 path uses the tcgen05 kernel in k_gemm_tc.cu instead.
#include "common.cuh"
#include "kernels.h"

namespace fm {

constexpr int SB_M = 64, SB_N = 64, SB_K = 16;

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  FM_PDL_ENTRY();
  __shared__ float As[SB_K][SB_M + 4];
  __shared__ float Bs[SB_K][SB_N + 4];
  const int b = blockIdx.z;
  const int m0 = blockIdx.y * SB_M, n0 = blockIdx.x * SB_N;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  const T* A = reinterpret_cast<const T*>(g.A) + (int64_t)b * g.sA;
  const T* B = reinterpret_cast<const T*>(g.B) + (int64_t)b * g.sB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += SB_K) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + 256 * i;
      int m, k;
      if (!g.a_mmajor) { m = e / SB_K; k = e % SB_K; } else { k = e / SB_M; m = e % SB_M; }
      int gm = m0 + m, gk = k0 + k;
      float v = 0.f;
      if (gm < g.M && gk < g.K)
        v = to_f<T>(g.a_mmajor ? A[(int64_t)gk * g.lda + gm] : A[(int64_t)gm * g.lda + gk]);
      As[k][m] = v;
      int n;
      if (!g.b_kmajor) { k = e / SB_N; n = e % SB_N; } else { n = e / SB_K; k = e % SB_K; }
      int gn = n0 + n;
      gk = k0 + k;
      v = 0.f;
      if (gn < g.N && gk < g.K)
        v = to_f<T>(g.b_kmajor ? B[(int64_t)gn * g.ldb + gk] : B[(int64_t)gk * g.ldb + gn]);
      Bs[k][n] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < SB_K; ++kk) {
      float a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int m = m0 + ty + 16 * i;
    if (m >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int n = n0 + tx + 16 * j;
      if (n >= g.N) continue;
      float v = acc[i][j] * g.alpha;
      if (g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32) {
        float* C = reinterpret_cast<float*>(g.C) + (int64_t)b * g.sC;
        if (g.epi == EPI_ACC_F32) C[(int64_t)m * g.ldc + n] += v;
        else C[(int64_t)m * g.ldc + n] = v;
        continue;
      }
      T* C = reinterpret_cast<T*>(g.C) + (int64_t)b * g.sC;
      if (g.bias) v += to_f<T>(reinterpret_cast<const T*>(g.bias)[(int64_t)b * g.sBias + n]);
      if (g.epi == EPI_STORE) {
        if (g.resid)
          v += to_f<T>(reinterpret_cast<const T*>(g.resid)[(int64_t)b * g.sR + (int64_t)m * g.ldr + n]);
        C[(int64_t)m * g.ldc + n] = from_f<T>(v);
      } else if (g.epi == EPI_BIAS_GELU_G) {
        T* D = reinterpret_cast<T*>(g.aux) + (int64_t)b * g.sAux;
        const float z = to_f<T>(from_f<T>(v));
        D[(int64_t)m * g.ldaux + n] = from_f<T>(gelu_grad_f(z));
        C[(int64_t)m * g.ldc + n] = from_f<T>(gelu_f(z));
      } else if (g.epi == EPI_MUL_AUX) {
        const T* D = reinterpret_cast<const T*>(g.aux) + (int64_t)b * g.sAux;
        C[(int64_t)m * g.ldc + n] = from_f<T>(v * to_f<T>(D[(int64_t)m * g.ldaux + n]));
      } else if (g.epi == EPI_BIAS_GELU) {
        T* Z = reinterpret_cast<T*>(g.aux) + (int64_t)b * g.sAux;
        T zq = from_f<T>(v);
        Z[(int64_t)m * g.ldaux + n] = zq;
        C[(int64_t)m * g.ldc + n] = from_f<T>(gelu_f(to_f<T>(zq)));
      } else {  // EPI_DGELU
        const T* Z = reinterpret_cast<const T*>(g.aux) + (int64_t)b * g.sAux;
        C[(int64_t)m * g.ldc + n] = from_f<T>(v * gelu_grad_f(to_f<T>(Z[(int64_t)m * g.ldaux + n])));
      }
    }
  }
}

int gemm_simt(const GemmArgs& g, int dtype, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return 0;
  dim3 grid((g.N + SB_N - 1) / SB_N, (g.M + SB_M - 1) / SB_M, g.batch);
  if (dtype == DT_F32) launch_k(gemm_simt_kernel<float>, grid, 256, 0, s, g);
  else launch_k(gemm_simt_kernel<bf16>, grid, 256, 0, s, g);
  return (int)cudaGetLastError();
}

int gemm(const GemmArgs& g, int dtype, cudaStream_t s) {
  if (dtype == DT_BF16) return gemm_tc(g, s);
  return gemm_simt(g, dtype, s);
}

}  // namespace fm
