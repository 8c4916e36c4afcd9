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
// 32*(w%4) .. +31, one output row per thread).  Persistent: grid = min(#tiles,
// #SMs), the smem ring runs across a CTA's tiles and the accumulator is double-
// buffered in TMEM so tile i's epilogue overlaps tile i+1's mainloop.
//
// Operand layouts (see kernels.h): A K-major [rows][K] or M-major [K][rows];
// B N-major [K][N] (weights W[in][out]) or K-major [N][K].  All tensors are
// described by 3-D TMA maps {inner, outer, batch}; out-of-bounds boxes are
// zero-filled by TMA, so ragged M/N/K tails need no special casing.
#include <cuda.h>
#include <stdio.h>
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace fm {

constexpr int TC_BM = 128, TC_BK = 64, TC_THREADS = 192;
static int g_tc_debug = 0;  // bit0: force SIMT for bf16; bit1: swap LBO/SBO of MN-major descs
static int g_force_bn = 0;  // 0 = wave-aware choice; 64/128/256 = forced tile width (benchmarks)
void gemm_tc_force_bn(int bn) { g_force_bn = bn; }
void gemm_tc_set_debug(int flags) { g_tc_debug = flags; }
int attn_tc_debug_off() { return g_tc_debug & 4; }  // bit2: force the SIMT attention kernels

// ------------------------------------------------------------ kernel
struct TcArgs {
  GemmArgs g;
  uint32_t idesc;
  int a_mmajor, b_kmajor, nk, dbg;
};

// Persistent: grid = min(#tiles, #SMs); CTA i walks tiles i, i + grid, ... (n fastest,
// then m, then batch).  The smem operand ring runs continuously across tiles, and the
// accumulator is double-buffered in TMEM (2 x BN columns) so the epilogue of tile i
// overlaps the TMA loads + MMAs of tile i+1.
template <int BN, int STAGES>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ CUtensorMap tma_c,
                   const __grid_constant__ CUtensorMap tma_aux, const TcArgs p) {
  constexpr uint32_t A_BYTES = TC_BM * TC_BK * 2;  // 16 KB
  constexpr uint32_t B_BYTES = BN * TC_BK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t RING = STAGES * STAGE_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const int ntn = (p.g.N + BN - 1) / BN, ntm = (p.g.M + TC_BM - 1) / TC_BM;
  const int num_tiles = ntn * ntm * p.g.batch;
  // one tile per CTA: the operand ring is free when the epilogue runs, so it doubles
  // as the staging area and a single TMEM accumulator suffices (smaller footprint)
  const bool single = num_tiles <= (int)gridDim.x;
  uint8_t* epi_smem = single ? smem : smem + RING;  // 4 epilogue warps x 2 x 4 KB staging
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING + (single ? 0 : 32768));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;      // [2] accumulator drained by the 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const GemmArgs& g = p.g;
  const uint32_t tmem_cols = single ? BN : 2 * BN;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 4); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  FM_PDL_ENTRY();

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer: one ring across all tiles of this CTA =====
      int gk = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int n0 = (tile % ntn) * BN, m0 = ((tile / ntn) % ntm) * TC_BM, b = tile / (ntn * ntm);
        for (int kb = 0; kb < p.nk; ++kb, ++gk) {
          const int s = gk % STAGES;
          if (gk >= STAGES) mbar_wait(&empty[s], ((gk / STAGES) + 1) & 1);
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
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer (one thread) =====
      const bool swap = (p.dbg & 2) != 0;
      const uint32_t mn_lbo = swap ? 1024u : 8192u, mn_sbo = swap ? 8192u : 1024u;
      int gk = 0, it = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
        const int acc = it & 1, use = it >> 1;
        if (use >= 1) mbar_wait(&tempty[acc], (use - 1) & 1);  // epilogue drained this buffer
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + acc * BN;
        for (int kb = 0; kb < p.nk; ++kb, ++gk) {
          const int s = gk % STAGES;
          mbar_wait(&full[s], (gk / STAGES) & 1);
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
            tc_mma(tmem_d, ad, bd, p.idesc, (kb > 0 || kk > 0) ? 1u : 0u);
          }
          tc_commit(&empty[s]);
        }
        tc_commit(&tfull[acc]);
      }
    }
  } else {
    // ===== epilogue: TMEM -> registers -> swizzled smem tile -> TMA store / reduce-add =====
    // Each warp owns 32 rows (its TMEM lane quarter) and walks the BN columns in
    // 32-column chunks.  A chunk is staged as a [32 rows][32 cols] box in smem with
    // the TMA swizzle (128 B rows for fp32, 64 B rows for bf16: conflict-free
    // 16-byte st.shared) and written by one TMA bulk store, or a TMA bulk
    // reduce-add (fp32 grad accumulation C += acc, done in L2).  Two staging
    // buffers per warp (4 KB each) overlap the next chunk with the in-flight store.
    const int quarter = warp & 3;
    const int r0 = quarter * 32;
    uint8_t* stage = epi_smem + quarter * 8192;
    const bool f32out = g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32;
    int buf = 0, it = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++it) {
      const int n0 = (tile % ntn) * BN, m0 = ((tile / ntn) % ntm) * TC_BM, b = tile / (ntn * ntm);
      const int acc = it & 1, use = it >> 1;
      const uint32_t tmem_acc = tmem_base + acc * BN;
      const int row = m0 + r0 + lane;
    const bool row_ok = row < g.M;
      // the per-row bf16 operand of the epilogue (Z for dGELU, the residual) is read
      // one 32-column chunk ahead, the first chunk before the accumulator is ready,
      // so its load latency hides under the mainloop / the previous chunk
      const bf16* xrow = nullptr;
      if (!f32out && row_ok) {
        if (g.epi == EPI_DGELU)
          xrow = reinterpret_cast<const bf16*>(g.aux) + (int64_t)b * g.sAux + (int64_t)row * g.ldaux;
        else if (g.epi == EPI_STORE && g.resid)
          xrow = reinterpret_cast<const bf16*>(g.resid) + (int64_t)b * g.sR + (int64_t)row * g.ldr;
      }
      uint4 pf[4];
      auto prefetch = [&](int c) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          pf[i] = (xrow && n0 + c + 8 * i < g.N) ? *reinterpret_cast<const uint4*>(xrow + n0 + c + 8 * i)
                                                   : make_uint4(0, 0, 0, 0);
      };
      prefetch(0);
      mbar_wait(&tfull[acc], use & 1);
      tc_fence_after();
#pragma unroll 1
    for (int c0 = 0; c0 < BN; c0 += 32) {
      const int nb = n0 + c0;
      if (nb >= g.N) break;  // warp-uniform
      float xv[32];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t w4[4] = {pf[i].x, pf[i].y, pf[i].z, pf[i].w};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          xv[8 * i + 2 * q] = __uint_as_float(w4[q] << 16);
          xv[8 * i + 2 * q + 1] = __uint_as_float(w4[q] & 0xFFFF0000u);
        }
      }
      if (c0 + 32 < BN) prefetch(c0 + 32);
      uint32_t r[32];
      tmem_ld32(tmem_acc + ((uint32_t)r0 << 16) + c0, r);
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * g.alpha;
      const int nvalid = min(32, g.N - nb);
      if (!f32out) {
        if (g.bias) {
          const bf16* bias = reinterpret_cast<const bf16*>(g.bias) + (int64_t)b * g.sBias + nb;
#pragma unroll
          for (int i = 0; i < 32; i += 8) {  // 16-byte loads (N % 8 == 0, so i < nvalid covers the group)
            float t[8];
            if (i < nvalid) load16<bf16>(bias + i, t);
#pragma unroll
            for (int q = 0; q < 8; ++q) v[i + q] += (i < nvalid) ? t[q] : 0.f;
          }
        }
        if (g.epi == EPI_STORE && g.resid && row_ok) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += xv[i];  // zeros past N
        } else if (g.epi == EPI_DGELU && row_ok) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= (i < nvalid) ? gelu_grad_f(xv[i]) : 0.f;
        }
      }
      // staging buffer `buf` is free once the store issued two chunks ago has read it
      if (lane == 0) bulk_wait_read<1>();
      __syncwarp();
      uint8_t* sb = stage + buf * 4096;
      if (f32out) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 q = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          *reinterpret_cast<float4*>(sb + lane * 128 + ((j ^ (lane & 7)) << 4)) = q;
        }
      } else if (g.epi == EPI_BIAS_GELU) {
        // aux = Z (pre-activation), C = GELU(bf16(Z))
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 zq, hq;
          float zz[8];
#pragma unroll
          for (int i = 0; i < 8; ++i) zz[i] = __bfloat162float(__float2bfloat16_rn(v[8 * j + i]));
          zq.x = pack_bf16x2(zz[0], zz[1]); zq.y = pack_bf16x2(zz[2], zz[3]);
          zq.z = pack_bf16x2(zz[4], zz[5]); zq.w = pack_bf16x2(zz[6], zz[7]);
          hq.x = pack_bf16x2(gelu_f(zz[0]), gelu_f(zz[1])); hq.y = pack_bf16x2(gelu_f(zz[2]), gelu_f(zz[3]));
          hq.z = pack_bf16x2(gelu_f(zz[4]), gelu_f(zz[5])); hq.w = pack_bf16x2(gelu_f(zz[6]), gelu_f(zz[7]));
          const int off = lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
          *reinterpret_cast<uint4*>(sb + off) = hq;
          *reinterpret_cast<uint4*>(sb + 2048 + off) = zq;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 q;
          q.x = pack_bf16x2(v[8 * j], v[8 * j + 1]); q.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
          q.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]); q.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
          *reinterpret_cast<uint4*>(sb + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) = q;
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        if (g.epi == EPI_ACC_F32) {
          tma_reduce_add_3d(&tma_c, sb, nb, m0 + r0, b);
        } else if (g.epi == EPI_STORE_F32) {
          tma_store_3d(&tma_c, sb, nb, m0 + r0, b);
        } else {
          tma_store_3d(&tma_c, sb, nb, m0 + r0, b);
          if (g.epi == EPI_BIAS_GELU) tma_store_3d(&tma_aux, sb + 2048, nb, m0 + r0, b);
        }
        bulk_commit();
      }
      buf ^= 1;
    }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);  // TMEM reads of this tile are complete
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem_base, tmem_cols);
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

// 3-D map {inner, outer, batch}; strides in elements; box {box_inner, box_outer, 1}.
static int make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer,
                    uint64_t batch, uint64_t ld, uint64_t bstride, uint32_t box_outer,
                    uint32_t box_inner = 64, bool f32 = false,
                    CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B) {
  const uint64_t es = f32 ? 4 : 2;
  cuuint64_t dims[3] = {inner, outer, batch};
  if (batch <= 1) bstride = ld * outer;
  cuuint64_t strides[2] = {ld * es, bstride * es};
  cuuint32_t box[3] = {box_inner, box_outer, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = g_encode(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3,
                        const_cast<void*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : (int)cudaErrorInvalidValue;
}

int make_tmap_2d_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld,
                      uint32_t box_inner, uint32_t box_outer) {
  if (int rc = gemm_tc_init()) return rc;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box,
                        estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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
  // output tiles: [32 rows][32 cols] boxes, fp32 (reduce-add, SW128) or bf16 (store, SW64)
  CUtensorMap mc, maux;
  const bool f32 = g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32;
  rc = make_map(&mc, g.C, g.N, g.M, g.batch, g.ldc, g.sC, 32, 32, f32,
                f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  maux = mc;
  if (g.epi == EPI_BIAS_GELU) {
    rc = make_map(&maux, g.aux, g.N, g.M, g.batch, g.ldaux, g.sAux, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
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
  const size_t smem_max = (size_t)STAGES * (TC_BM * TC_BK * 2 + BN * TC_BK * 2) + 32768 + 1024 + 256;
  auto kern = gemm_tc_kernel<BN, STAGES>;
  static bool attr_set = (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max), true);
  (void)attr_set;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  const int64_t tiles = (int64_t)((g.N + BN - 1) / BN) * ((g.M + TC_BM - 1) / TC_BM) * g.batch;
  const int grid = (int)(tiles < num_sms ? tiles : num_sms);
  const size_t smem = tiles <= grid ? smem_max - 32768 : smem_max;
  launch_k(kern, dim3(grid), TC_THREADS, smem, s, ma, mb, mc, maux, p);
  return (int)cudaGetLastError();
}

int gemm_tc(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0 || g.K <= 0) return 0;
  if (g_tc_debug & 1) return gemm_simt(g, DT_BF16, s);
  if (int rc = gemm_tc_init()) return rc;
  // Tile width (measured, tools/gemm_microbench.py): BN=256 (best MMA/operand efficiency)
  // whenever it still yields >= 48 tiles; small, latency-bound GEMMs get narrower tiles
  // and more CTAs.
  if (g_force_bn == 256) return launch_tc<256, 4>(g, s);
  if (g_force_bn == 128) return launch_tc<128, 6>(g, s);
  if (g_force_bn == 64) return launch_tc<64, 8>(g, s);
  const int64_t mt = (int64_t)((g.M + TC_BM - 1) / TC_BM) * g.batch;
  auto tiles = [&](int bn) { return mt * ((g.N + bn - 1) / bn); };
  if (g.N >= 256 && tiles(256) >= 48) return launch_tc<256, 4>(g, s);
  if (g.N >= 128 && tiles(128) >= 48) return launch_tc<128, 6>(g, s);
  return launch_tc<64, 8>(g, s);
}

}  // namespace fm
