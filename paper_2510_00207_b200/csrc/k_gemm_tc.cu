// K4/K5 gemm_tc: bf16 x bf16 -> fp32 (TMEM) GEMM on the 5th-generation tensor
// cores (tcgen05.mma, cta_group::1), operands staged by TMA (128-byte swizzle)
// through a multi-stage mbarrier ring, accumulator in TMEM, fused epilogues
// (bias, GELU with pre-activation save, GELU' for dgrad, residual add, fp32
// grad accumulation).  Serves every dense contraction of the FlowMoE block:
// the MHA projections (S1/S3, B5), and the batched expert GEMMs (S7, B2) whose
// rows are the capacity-padded [E/P][P·C] buffers (uniform shapes => batched).
//
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// single-thread MMA issuer, warps 2..5 = epilogue (warp w reads TMEM lanes
// 32*(w%4) .. +31, one output row per thread).
//
// Operand layouts (see kernels.h): A K-major [rows][K] or M-major [K][rows];
// B N-major [K][N] (weights W[in][out]) or K-major [N][K].  All tensors are
// described by 3-D TMA maps {inner, outer, batch}; out-of-bounds boxes are
// zero-filled by TMA, so ragged M/N/K tails need no special casing.
#include <cuda.h>
#include <stdio.h>
#include "common.cuh"
#include "kernels.h"

namespace fm {

constexpr int TC_BM = 128, TC_BK = 64, TC_THREADS = 192;
static int g_tc_debug = 0;  // bit0: force SIMT for bf16; bit1: swap LBO/SBO of MN-major descs
void gemm_tc_set_debug(int flags) { g_tc_debug = flags; }

// ------------------------------------------------------------ PTX wrappers
FM_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

FM_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
FM_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
FM_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } while (!ok);
}
FM_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}
FM_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
FM_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
FM_DEV void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
FM_DEV void tc_mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                   uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
FM_DEV void tmem_ld32(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// UMMA shared-memory descriptor (SWIZZLE_128B, version 1 for sm_100).
FM_DEV uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (Blackwell)
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

// ------------------------------------------------------------ kernel
struct TcArgs {
  GemmArgs g;
  uint32_t idesc;
  int a_mmajor, b_kmajor, nk, dbg;
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b, const TcArgs p) {
  constexpr uint32_t A_BYTES = TC_BM * TC_BK * 2;  // 16 KB
  constexpr uint32_t B_BYTES = BN * TC_BK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN, m0 = blockIdx.y * TC_BM, b = blockIdx.z;
  const GemmArgs& g = p.g;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"((uint32_t)BN));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      for (int kb = 0; kb < p.nk; ++kb) {
        const int s = kb % STAGES;
        if (kb >= STAGES) mbar_wait(&empty[s], ((kb / STAGES) + 1) & 1);
        uint8_t* sa = smem + s * STAGE_BYTES;
        uint8_t* sb = sa + A_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        const int k0 = kb * TC_BK;
        if (!p.a_mmajor) {
          tma_load_3d(sa, &tma_a, &full[s], k0, m0, b);
        } else {
#pragma unroll
          for (int i = 0; i < TC_BM / 64; ++i) tma_load_3d(sa + i * 8192, &tma_a, &full[s], m0 + 64 * i, k0, b);
        }
        if (p.b_kmajor) {
          tma_load_3d(sb, &tma_b, &full[s], k0, n0, b);
        } else {
#pragma unroll
          for (int i = 0; i < BN / 64; ++i) tma_load_3d(sb + i * 8192, &tma_b, &full[s], n0 + 64 * i, k0, b);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (one thread) =====
      const bool swap = (p.dbg & 2) != 0;
      const uint32_t mn_lbo = swap ? 1024u : 8192u, mn_sbo = swap ? 8192u : 1024u;
      for (int kb = 0; kb < p.nk; ++kb) {
        const int s = kb % STAGES;
        mbar_wait(&full[s], (kb / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * STAGE_BYTES);
        const uint32_t sb = sa + A_BYTES;
#pragma unroll
        for (int kk = 0; kk < TC_BK / 16; ++kk) {
          // K-major: +32 B per UMMA_K=16 inside the 128-B swizzle row; SBO = 8 rows * 128 B.
          // MN-major: +16 K-rows * 128 B; LBO = 64-element MN block stride (one TMA box).
          const uint64_t ad = p.a_mmajor ? umma_desc(sa + kk * 2048, mn_lbo, mn_sbo)
                                         : umma_desc(sa + kk * 32, 16, 1024);
          const uint64_t bd = p.b_kmajor ? umma_desc(sb + kk * 32, 16, 1024)
                                         : umma_desc(sb + kk * 2048, mn_lbo, mn_sbo);
          tc_mma(tmem_base, ad, bd, p.idesc, (kb > 0 || kk > 0) ? 1u : 0u);
        }
        tc_commit(&empty[s]);
      }
      tc_commit(tmem_full);
    }
  } else {
    // ===== epilogue: TMEM -> registers -> global =====
    const int quarter = warp & 3;
    const int row = m0 + quarter * 32 + lane;
    mbar_wait(tmem_full, 0);
    tc_fence_after();
    const bool row_ok = row < g.M;
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      uint32_t r[32];
      tmem_ld32(tmem_base + ((uint32_t)(quarter * 32) << 16) + c0, r);
      const int nb = n0 + c0;
      if (!row_ok || nb >= g.N) continue;
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * g.alpha;
      const int nvalid = min(32, g.N - nb);
      if (g.epi == EPI_ACC_F32) {
        float* C = reinterpret_cast<float*>(g.C) + (int64_t)b * g.sC + (int64_t)row * g.ldc + nb;
        if (nvalid == 32) {
#pragma unroll
          for (int i = 0; i < 32; i += 4) {
            float4 o = *reinterpret_cast<float4*>(C + i);
            o.x += v[i]; o.y += v[i + 1]; o.z += v[i + 2]; o.w += v[i + 3];
            *reinterpret_cast<float4*>(C + i) = o;
          }
        } else {
          for (int i = 0; i < nvalid; ++i) C[i] += v[i];
        }
        continue;
      }
      if (g.bias) {
        const bf16* bias = reinterpret_cast<const bf16*>(g.bias) + (int64_t)b * g.sBias + nb;
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] += (i < nvalid) ? __bfloat162float(bias[i]) : 0.f;
      }
      bf16* C = reinterpret_cast<bf16*>(g.C) + (int64_t)b * g.sC + (int64_t)row * g.ldc + nb;
      if (g.epi == EPI_STORE) {
        if (g.resid) {
          const bf16* R = reinterpret_cast<const bf16*>(g.resid) + (int64_t)b * g.sR + (int64_t)row * g.ldr + nb;
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += (i < nvalid) ? __bfloat162float(R[i]) : 0.f;
        }
      } else if (g.epi == EPI_BIAS_GELU) {
        bf16* Z = reinterpret_cast<bf16*>(g.aux) + (int64_t)b * g.sAux + (int64_t)row * g.ldaux + nb;
        if (nvalid == 32) {
#pragma unroll
          for (int i = 0; i < 32; i += 8) store16<bf16>(Z + i, v + i);
        } else {
          for (int i = 0; i < nvalid; ++i) Z[i] = __float2bfloat16_rn(v[i]);
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = gelu_f(__bfloat162float(__float2bfloat16_rn(v[i])));
      } else {  // EPI_DGELU
        const bf16* Z = reinterpret_cast<const bf16*>(g.aux) + (int64_t)b * g.sAux + (int64_t)row * g.ldaux + nb;
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] *= (i < nvalid) ? gelu_grad_f(__bfloat162float(Z[i])) : 0.f;
      }
      if (nvalid == 32) {
#pragma unroll
        for (int i = 0; i < 32; i += 8) store16<bf16>(C + i, v + i);
      } else {
        for (int i = 0; i < nvalid; ++i) C[i] = __float2bfloat16_rn(v[i]);
      }
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"((uint32_t)BN));
  }
}

// ------------------------------------------------------------ host side
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static PFN_encodeTiled g_encode = nullptr;

int gemm_tc_init() {
  if (g_encode) return 0;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || fn == nullptr) return (int)(e ? e : cudaErrorNotSupported);
  g_encode = reinterpret_cast<PFN_encodeTiled>(fn);
  return 0;
}

// 3-D bf16 map {inner, outer, batch}; strides in elements; box {64, box_outer, 1}.
static int make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                    uint64_t batch, uint64_t ld, uint64_t bstride, uint32_t box_outer) {
  cuuint64_t dims[3] = {inner, outer, batch};
  if (batch <= 1) bstride = ld * outer;
  cuuint64_t strides[2] = {ld * 2, bstride * 2};
  cuuint32_t box[3] = {64, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

template <int BN, int STAGES>
static int launch_tc(const GemmArgs& g, cudaStream_t s) {
  CUtensorMap ma, mb;
  int rc;
  if (!g.a_mmajor) rc = make_map(&ma, g.A, g.K, g.M, g.batch, g.lda, g.sA, TC_BM);
  else rc = make_map(&ma, g.A, g.M, g.K, g.batch, g.lda, g.sA, TC_BK);
  if (rc) return rc;
  if (g.b_kmajor) rc = make_map(&mb, g.B, g.K, g.N, g.batch, g.ldb, g.sB, BN);
  else rc = make_map(&mb, g.B, g.N, g.K, g.batch, g.ldb, g.sB, TC_BK);
  if (rc) return rc;
  TcArgs p;
  p.g = g;
  p.a_mmajor = g.a_mmajor;
  p.b_kmajor = g.b_kmajor;
  p.nk = (g.K + TC_BK - 1) / TC_BK;
  p.dbg = g_tc_debug;
  // kind::f16 instruction descriptor: D f32, A/B bf16, majors, N>>3, M>>4
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(g.a_mmajor ? 1 : 0) << 15) |
            ((uint32_t)(g.b_kmajor ? 0 : 1) << 16) | ((uint32_t)(BN >> 3) << 17) |
            ((uint32_t)(TC_BM >> 4) << 24);
  const size_t smem = (size_t)STAGES * (TC_BM * TC_BK * 2 + BN * TC_BK * 2) + 1024 + 256;
  auto kern = gemm_tc_kernel<BN, STAGES>;
  static bool attr_set = (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), true);
  (void)attr_set;
  dim3 grid((g.N + BN - 1) / BN, (g.M + TC_BM - 1) / TC_BM, g.batch);
  kern<<<grid, TC_THREADS, smem, s>>>(ma, mb, p);
  return (int)cudaGetLastError();
}

int gemm_tc(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0 || g.K <= 0) return 0;
  if (g_tc_debug & 1) return gemm_simt(g, DT_BF16, s);
  if (int rc = gemm_tc_init()) return rc;
  if (g.N >= 256) return launch_tc<256, 4>(g, s);
  if (g.N >= 128) return launch_tc<128, 6>(g, s);
  return launch_tc<64, 8>(g, s);
}

}  // namespace fm
