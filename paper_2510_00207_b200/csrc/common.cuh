// Shared device helpers for the FlowMoE B200 kernels (sm_100a only).
// No code here is shared with oracle/ (the CPU checker); see DESIGN.md.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <utility>

#define FM_DEV __device__ __forceinline__

namespace fm {

typedef __nv_bfloat16 bf16;

// ---- element conversion (storage dtype <-> fp32 math) ----
template <typename T> FM_DEV float to_f(T v);
template <> FM_DEV float to_f<float>(float v) { return v; }
template <> FM_DEV float to_f<bf16>(bf16 v) { return __bfloat162float(v); }
template <typename T> FM_DEV T from_f(float v);
template <> FM_DEV float from_f<float>(float v) { return v; }
template <> FM_DEV bf16 from_f<bf16>(float v) { return __float2bfloat16_rn(v); }

// 16-byte vector of storage elements: 4 floats or 8 bf16.
template <typename T> struct Vec16 { static constexpr int N = 16 / sizeof(T); };

template <typename T>
FM_DEV void load16(const T* p, float* out) {
  uint4 u = *reinterpret_cast<const uint4*>(p);
  if constexpr (sizeof(T) == 4) {
    out[0] = __uint_as_float(u.x); out[1] = __uint_as_float(u.y);
    out[2] = __uint_as_float(u.z); out[3] = __uint_as_float(u.w);
  } else {
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      out[2 * i] = __uint_as_float(w[i] << 16);
      out[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
    }
  }
}

FM_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <typename T>
FM_DEV void store16(T* p, const float* in) {
  uint4 u;
  if constexpr (sizeof(T) == 4) {
    u.x = __float_as_uint(in[0]); u.y = __float_as_uint(in[1]);
    u.z = __float_as_uint(in[2]); u.w = __float_as_uint(in[3]);
  } else {
    u.x = pack_bf16x2(in[0], in[1]); u.y = pack_bf16x2(in[2], in[3]);
    u.z = pack_bf16x2(in[4], in[5]); u.w = pack_bf16x2(in[6], in[7]);
  }
  *reinterpret_cast<uint4*>(p) = u;
}

FM_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
FM_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// GELU with erf (reading Q8) and its derivative.
FM_DEV float gelu_f(float z) { return 0.5f * z * (1.0f + erff(z * 0.70710678118654752f)); }
FM_DEV float gelu_grad_f(float z) {
  return 0.5f * (1.0f + erff(z * 0.70710678118654752f)) +
         z * __expf(-0.5f * z * z) * 0.39894228040143268f;
}

// ---- programmatic dependent launch (PDL) ----
// Every kernel is launched with programmatic stream serialization, so it may be
// scheduled while its predecessor on the stream is still running.  Each kernel
// therefore calls griddep_wait() before its first global-memory access (after its
// smem/TMEM/barrier prologue in the tensor-core kernels), which blocks until the
// predecessor grid has completed and flushed; it then calls griddep_launch() so
// the successor's prologue can overlap this kernel's body.
FM_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
FM_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }
#define FM_PDL_ENTRY() \
  do {                 \
    fm::griddep_wait();  \
    fm::griddep_launch(); \
  } while (0)

extern int g_pdl_enabled;  // flowmoe_debug_set(4, 0) turns PDL off (A/B measurements)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl_enabled;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

// launch_k with a thread-block cluster shape (DSMEM reductions across the cluster)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_kc(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             dim3 cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = g_pdl_enabled;
  at[1].id = cudaLaunchAttributeClusterDimension;
  at[1].val.clusterDim.x = cluster.x;
  at[1].val.clusterDim.y = cluster.y;
  at[1].val.clusterDim.z = cluster.z;
  cfg.attrs = at;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

}  // namespace fm
