// Optimizer step over contiguous fp32 master weights (reading Q17: the paper updates
// the experts as soon as their gradients are final, without naming the
// optimizer): SGD with momentum + L2 decay, or AdamW (decoupled decay).  Writes the
// master, the state and, if given, the compute copy in the config dtype.  HBM-bound:
// 16-byte vectors, grid-stride; scalar path for unaligned tensors.
#include "common.cuh"
#include "kernels.h"

namespace fm {

struct OptArgs {
  float lr, b1, b2, eps, wd, bc1, bc2;  // bc = 1 - beta^step (AdamW bias corrections)
  int first;                            // SGD: step 1 initialises the momentum buffer
};

template <int KIND>
FM_DEV float opt_elem(float& w, float& s1, float& s2, float g, const OptArgs& a) {
  if (KIND == 0) {  // SGD-momentum: d = g + wd·w; b = μ·b + d (b = d at step 1); w -= lr·b
    const float d = g + a.wd * w;
    s1 = a.first ? d : a.b1 * s1 + d;
    w -= a.lr * s1;
  } else {          // AdamW
    s1 = a.b1 * s1 + (1.f - a.b1) * g;
    s2 = a.b2 * s2 + (1.f - a.b2) * g * g;
    const float mh = s1 / a.bc1, vh = s2 / a.bc2;
    w = w * (1.f - a.lr * a.wd) - a.lr * mh / (sqrtf(vh) + a.eps);
  }
  return w;
}

template <typename T, int KIND, bool VEC>
__global__ void __launch_bounds__(256) optim_kernel(float* w, float* s1, float* s2, const float* g, T* out,
                                                    int64_t n, OptArgs a) {
  FM_PDL_ENTRY();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (VEC) {
    const int64_t nv = n / 4;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nv; i += stride) {
      float4 wv = reinterpret_cast<float4*>(w)[i], gv = reinterpret_cast<const float4*>(g)[i];
      float4 av = reinterpret_cast<float4*>(s1)[i];
      float4 bv = KIND == 1 ? reinterpret_cast<float4*>(s2)[i] : make_float4(0.f, 0.f, 0.f, 0.f);
      float r[4];
      r[0] = opt_elem<KIND>(wv.x, av.x, bv.x, gv.x, a);
      r[1] = opt_elem<KIND>(wv.y, av.y, bv.y, gv.y, a);
      r[2] = opt_elem<KIND>(wv.z, av.z, bv.z, gv.z, a);
      r[3] = opt_elem<KIND>(wv.w, av.w, bv.w, gv.w, a);
      reinterpret_cast<float4*>(w)[i] = wv;
      reinterpret_cast<float4*>(s1)[i] = av;
      if (KIND == 1) reinterpret_cast<float4*>(s2)[i] = bv;
      if (out)
#pragma unroll
        for (int q = 0; q < 4; ++q) out[4 * i + q] = from_f<T>(r[q]);
    }
    for (int64_t i = nv * 4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      float z = 0.f;
      const float r = opt_elem<KIND>(w[i], s1[i], KIND == 1 ? s2[i] : z, g[i], a);
      if (out) out[i] = from_f<T>(r);
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
      float z = 0.f;
      const float r = opt_elem<KIND>(w[i], s1[i], KIND == 1 ? s2[i] : z, g[i], a);
      if (out) out[i] = from_f<T>(r);
    }
  }
}

template <typename T, int KIND>
static void optim_launch(float* w, float* s1, float* s2, const float* g, void* out, int64_t n, const OptArgs& a,
                         cudaStream_t s) {
  int64_t blocks = (n / 4 + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 8) blocks = 148 * 8;
  const bool vec = ((reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(s1) |
                     reinterpret_cast<uintptr_t>(g) | (KIND == 1 ? reinterpret_cast<uintptr_t>(s2) : 0)) & 15) == 0;
  if (vec)
    launch_k(optim_kernel<T, KIND, true>, dim3((unsigned)blocks), 256, 0, s, w, s1, s2, g, (T*)out, n, a);
  else
    launch_k(optim_kernel<T, KIND, false>, dim3((unsigned)blocks), 256, 0, s, w, s1, s2, g, (T*)out, n, a);
}

int optim_step(int dtype, int kind, float lr, float b1, float b2, float eps, float wd, int64_t step, float* w,
               float* s1, float* s2, const float* g, void* out, int64_t n, cudaStream_t s) {
  if (n <= 0) return 0;
  OptArgs a;
  a.lr = lr; a.b1 = b1; a.b2 = b2; a.eps = eps; a.wd = wd;
  a.bc1 = (float)(1.0 - pow((double)b1, (double)step));
  a.bc2 = (float)(1.0 - pow((double)b2, (double)step));
  a.first = step == 1;
  if (kind == 0) {
    if (dtype == DT_F32) optim_launch<float, 0>(w, s1, s2, g, out, n, a, s);
    else optim_launch<bf16, 0>(w, s1, s2, g, out, n, a, s);
  } else {
    if (dtype == DT_F32) optim_launch<float, 1>(w, s1, s2, g, out, n, a, s);
    else optim_launch<bf16, 1>(w, s1, s2, g, out, n, a, s);
  }
  return (int)cudaGetLastError();
}

}  // namespace fm
