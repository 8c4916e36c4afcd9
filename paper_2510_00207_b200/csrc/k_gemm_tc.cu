// K4/K5 gemm_tc: bf16 x bf16 -> fp32 (TMEM) GEMM on the 5th-generation tensor
// cores (tcgen05.mma, cta_group::1), operands staged by TMA (128-byte swizzle)
// through a multi-stage mbarrier ring, accumulator in TMEM, fused epilogues
// (bias, GELU with pre-activation save, GELU' for dgrad, residual add, fp32
// grad accumulation).  Serves every dense contraction of the FlowMoE block:
// the MHA projections (S1/S3, B5), and the batched expert GEMMs (S7, B2) whose
// rows are the capacity-padded [E/P][P·C] buffers (uniform shapes => batched).
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer (one elected lane), warps 2..9 = epilogue (warp w reads TMEM lanes
// 32*(w%4) .. +31, one output row per thread, alternate 32-column chunks).  Persistent: grid = min(#tiles,
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

constexpr int TC_BM = 128, TC_BK = 64, TC_THREADS = 320;  // producer, MMA, 8 epilogue warps

// Phase probe (tools/probe/gemm_probe.cu builds this file with -DFM_PROBE): SM clock
// stamps of CTA 0's phases.  Compiled out of the library.
#ifdef FM_PROBE
__device__ long long g_probe[32];
#define FM_MARK(i) do { if (blockIdx.x == 0) g_probe[i] = clock64(); } while (0)
#else
#define FM_MARK(i) do {} while (0)
#endif
static int g_tc_debug = 0;  // bit0: force SIMT for bf16; bit1: swap LBO/SBO of MN-major descs
static int g_force_bn = 0;  // 0 = wave-aware choice; 64/128/256 = forced tile width (benchmarks)
static int g_force_cg = 0;  // 0 = automatic; 1 = one CTA per tile; 2 = CTA pair (cta_group::2)
void gemm_tc_force_bn(int bn) { g_force_bn = bn; }
void gemm_tc_force_cg(int cg) { g_force_cg = cg; }
static int g_force_sk = 0;  // stream-K: 0 = automatic, 1 = never, 2 = wherever the scratch allows
void gemm_tc_force_streamk(int mode) { g_force_sk = mode; }
void gemm_tc_set_debug(int flags) { g_tc_debug = flags; }
int attn_tc_debug_off() { return g_tc_debug & 4; }  // bit2: force the SIMT attention kernels

// ------------------------------------------------------------ kernel
struct TcArgs {
  GemmArgs g;
  uint32_t idesc;
  int a_mmajor, b_kmajor, nk, dbg;
  int streamk;  // 1: stream-K work split (g.splitk_ws / g.splitk_tick hold the fix-up state)
};

// Persistent: grid = min(#tiles, #SMs) units; unit i walks tiles i, i + #units, ... (n
// fastest, then m, then batch).  The smem operand ring runs continuously across tiles,
// and the accumulator is double-buffered in TMEM (2 x BN columns) so the epilogue of tile
// i overlaps the TMA loads + MMAs of tile i+1.
// CG = 2: a unit is a CTA pair (cluster of 2 on one TPC) running M = 256 UMMAs
// (tcgen05.mma.cta_group::2, issued by the leader CTA): each CTA loads its own 128 rows of
// A and half (BN/2) of the B columns and gets its 128 accumulator rows in its own TMEM, so
// the operand bytes per SM and K-step drop from (128 + BN)·BK·2 to (128 + BN/2)·BK·2 —
// the L2->SMEM traffic that bounded the 1-CTA kernel at ~70% of the tensor peak.
template <int BN, int STAGES, int EB, int CG, bool SK>
__global__ void __launch_bounds__(TC_THREADS, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma_a,
                   const __grid_constant__ CUtensorMap tma_b,
                   const __grid_constant__ CUtensorMap tma_c,
                   const __grid_constant__ CUtensorMap tma_aux, const TcArgs p) {
  constexpr int BNL = BN / CG;                      // B columns this CTA loads
  // pair tiles wider than one UMMA (BN = 512, CG = 2): NSUB UMMAs of N = UN per K-step share
  // the A operand; the CTA loads SUBL columns of each UMMA's B; the accumulator then fills
  // TMEM (one buffer: the next tile's MMAs wait for the epilogue to drain it)
  constexpr int NSUB = (CG == 2 && BN > 256) ? BN / 256 : 1;
  constexpr int UN = BN / NSUB, SUBL = UN / CG;
  constexpr int NACC = 2 * BN <= 512 ? 2 : 1;
  constexpr uint32_t A_BYTES = TC_BM * TC_BK * 2;  // 16 KB
  constexpr uint32_t B_BYTES = BNL * TC_BK * 2;
  constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  constexpr uint32_t RING = STAGES * STAGE_BYTES;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t crank = CG == 2 ? cluster_rank() : 0u;
  const bool leader = crank == 0;
  const int unit = (int)blockIdx.x / CG, nunits = (int)gridDim.x / CG;
  const int ntn = (p.g.N + BN - 1) / BN, ntm = (p.g.M + TC_BM * CG - 1) / (TC_BM * CG);
  const int num_tiles = ntn * ntm * p.g.batch;
  // Work split.  Whole tiles: unit u takes tiles u, u + #units, ...  Stream-K (SK): the
  // tiles of the full waves stay whole (data-parallel), and the k-blocks of the remaining
  // tiles (fewer than #units), flattened in (tile, k-block) order, are cut into #units
  // equal ranges, one per unit after its whole tiles: every SM (pair) gets the same work
  // however the tiles quantise.  A "segment" is one unit's k-block range [kb0, kb1) of one
  // tile; the segments of a cut tile are summed by the epilogue's fix-up.
  constexpr bool sk = SK;  // compiled out of the whole-tile instantiations (register budget)
  const int dp_tiles = sk ? num_tiles / nunits * nunits : num_tiles;
  const int64_t sk_base = (int64_t)dp_tiles * p.nk, sk_total = (int64_t)num_tiles * p.nk - sk_base;
  const int64_t sk_b = sk_base + (int64_t)unit * sk_total / nunits;
  const int64_t sk_e = sk_base + (int64_t)(unit + 1) * sk_total / nunits;
  const int64_t it_begin = unit < dp_tiles ? (int64_t)unit * p.nk : sk_b;
  auto seg_more = [&](int64_t w) { return w < sk_base || w < sk_e; };
  auto seg_of = [&](int64_t w, int& tile, int& kb0, int& kb1) {
    tile = (int)(w / p.nk);
    kb0 = (int)(w - (int64_t)tile * p.nk);
    kb1 = (!sk || w < sk_base) ? p.nk : (int)min((int64_t)p.nk, (int64_t)kb0 + (sk_e - w));
  };
  auto seg_next = [&](int64_t w, int tile, int kb0, int kb1) -> int64_t {
    if (w < sk_base) return tile + nunits < dp_tiles ? (int64_t)(tile + nunits) * p.nk : sk_b;
    return w + (kb1 - kb0);
  };
  // one tile per unit: the operand ring is free when the epilogue runs, so it doubles
  // as the staging area and a single TMEM accumulator suffices (smaller footprint)
  const bool single = !sk && num_tiles <= nunits;
  uint8_t* epi_smem = single ? smem : smem + RING;  // 8 epilogue warps x EB x 4 KB staging
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + RING + (single ? 0 : EB * 32768));
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;  // [2] accumulator ready
  uint64_t* tempty = tfull + 2;      // [2] accumulator drained by the 4 epilogue warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const GemmArgs& g = p.g;
  // TMEM allocations are powers of two >= 32 columns (BN = 192: 256 / 512)
  const uint32_t tmem_cols = single ? (BN <= 64 ? 64u : BN <= 128 ? 128u : BN <= 256 ? 256u : 512u)
                                    : (NACC * BN <= 128 ? 128u : NACC * BN <= 256 ? 256u : 512u);
  if (threadIdx.x == 0) FM_MARK(0);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int a = 0; a < 2; ++a) { mbar_init(&tfull[a], 1); mbar_init(&tempty[a], 8 * CG); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tma_b)) : "memory");
  }
  if (warp == 1) {
    if constexpr (CG == 2) tmem_alloc2(tmem_slot, tmem_cols);
    else tmem_alloc(tmem_slot, tmem_cols);
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) cluster_sync_all();  // both CTAs' barriers initialised before any remote use
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  if (threadIdx.x == 0) FM_MARK(1);
  FM_PDL_ENTRY();
  if (threadIdx.x == 0) FM_MARK(2);

  if (warp == 0) {
    // ===== TMA producer (whole warp walks the ring, one elected lane issues) =====
    int gk = 0;
    for (int64_t w = it_begin; seg_more(w);) {
      int tile, kb0, kb1;
      seg_of(w, tile, kb0, kb1);
      w = seg_next(w, tile, kb0, kb1);
      const int n0 = (tile % ntn) * BN + (int)crank * SUBL;  // this CTA's B columns (+ s·UN per UMMA)
      const int m0 = ((tile / ntn) % ntm) * TC_BM * CG + (int)crank * TC_BM, b = tile / (ntn * ntm);
      for (int kb = kb0; kb < kb1; ++kb, ++gk) {
        const int s = gk % STAGES;
        if (gk >= STAGES) {
          if constexpr (CG == 2) mbar_wait_cl(&empty[s], ((gk / STAGES) + 1) & 1);
          else mbar_wait(&empty[s], ((gk / STAGES) + 1) & 1);
        }
        uint8_t* sa = smem + s * STAGE_BYTES;
        uint8_t* sb = sa + A_BYTES;
        const int k0 = kb * TC_BK;
        if (elect_one()) {
          if constexpr (CG == 1) {
            mbar_expect_tx(&full[s], STAGE_BYTES);
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
              for (int i = 0; i < BNL / 64; ++i) tma_load_3d(sb + i * 8192, &tma_b, &full[s], n0 + 64 * i, k0, b);
            }
          } else {
            // both CTAs' bytes complete on the leader's barrier, armed by the leader alone
            if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
            const uint32_t bar = mapa_u32(smem_u32(&full[s]), 0);
            if (!p.a_mmajor) {
              tma_load_3d_cg2(sa, &tma_a, bar, k0, m0, b);
            } else {
#pragma unroll
              for (int i = 0; i < TC_BM / 64; ++i) tma_load_3d_cg2(sa + i * 8192, &tma_a, bar, m0 + 64 * i, k0, b);
            }
#pragma unroll
            for (int u = 0; u < NSUB; ++u) {
              uint8_t* sbu = sb + u * SUBL * TC_BK * 2;
              if (p.b_kmajor) {
                tma_load_3d_cg2(sbu, &tma_b, bar, k0, n0 + u * UN, b);
              } else {
#pragma unroll
                for (int i = 0; i < SUBL / 64; ++i)
                  tma_load_3d_cg2(sbu + i * 8192, &tma_b, bar, n0 + u * UN + 64 * i, k0, b);
              }
            }
          }
          if (gk < 4) FM_MARK(24 + gk);
        }
        __syncwarp();
      }
    }
    if constexpr (CG == 2) {
      // drain: every stage's last release (the leader's multicast commit) has landed in this
      // CTA's smem before the pair may exit
      for (int q = gk - STAGES; q < gk; ++q)  // release of use q / STAGES = that phase's completion
        if (q >= 0) mbar_wait_cl(&empty[q % STAGES], (q / STAGES) & 1);
    }
  } else if (warp == 1 && (CG == 1 || leader)) {
    // ===== MMA issuer (whole warp waits, one elected lane issues; the pair's leader) =====
    const bool swap = (p.dbg & 2) != 0;
    const uint32_t mn_lbo = swap ? 1024u : 8192u, mn_sbo = swap ? 8192u : 1024u;
    // Descriptors of stage 0 built once; a stage / UMMA_K step only adds to the 14-bit
    // start-address field (smem < 256 KB, so no carry out of it).
    // K-major: +32 B per UMMA_K=16 inside the 128-B swizzle row; SBO = 8 rows * 128 B.
    // MN-major: +16 K-rows * 128 B; LBO = 64-element MN block stride (one TMA box).
    const uint32_t s0 = smem_u32(smem);
    const uint64_t adesc0 = p.a_mmajor ? umma_desc(s0, mn_lbo, mn_sbo) : umma_desc(s0, 16, 1024);
    const uint64_t bdesc0 = p.b_kmajor ? umma_desc(s0 + A_BYTES, 16, 1024) : umma_desc(s0 + A_BYTES, mn_lbo, mn_sbo);
    const uint64_t a_kstep = p.a_mmajor ? (2048 >> 4) : (32 >> 4);
    const uint64_t b_kstep = p.b_kmajor ? (32 >> 4) : (2048 >> 4);
    int gk = 0, it = 0;
    for (int64_t w = it_begin; seg_more(w); ++it) {
      int tile, kb0, kb1;
      seg_of(w, tile, kb0, kb1);
      w = seg_next(w, tile, kb0, kb1);
      const int acc = NACC == 2 ? (it & 1) : 0, use = NACC == 2 ? (it >> 1) : it;
      if (use >= 1) {  // the epilogue(s) drained this buffer
        if constexpr (CG == 2) mbar_wait_cl(&tempty[acc], (use - 1) & 1);
        else mbar_wait(&tempty[acc], (use - 1) & 1);
      }
      tc_fence_after();
      const uint32_t tmem_d = tmem_base + acc * BN;
      (void)tile;
      for (int kb = kb0; kb < kb1; ++kb, ++gk) {
        const int s = gk % STAGES;
        if constexpr (CG == 2) mbar_wait_cl(&full[s], (gk / STAGES) & 1);
        else mbar_wait(&full[s], (gk / STAGES) & 1);
        if (lane == 0 && gk == 0) FM_MARK(3);
        if (lane == 0 && gk < 8) FM_MARK(16 + gk);
        tc_fence_after();
        const uint64_t soff = (uint64_t)((uint32_t)s * STAGE_BYTES >> 4);
        if (elect_one()) {
#pragma unroll
          for (int kk = 0; kk < TC_BK / 16; ++kk) {
            if constexpr (CG == 2) {
#pragma unroll
              for (int u = 0; u < NSUB; ++u)  // B of UMMA u: SUBL rows (K-major) / columns further on
                tc_mma2(tmem_d + u * UN, adesc0 + soff + kk * a_kstep,
                        bdesc0 + soff + kk * b_kstep + (uint64_t)(u * SUBL * TC_BK * 2 >> 4), p.idesc,
                        (kb > kb0 || kk > 0) ? 1u : 0u);
            } else
              tc_mma(tmem_d, adesc0 + soff + kk * a_kstep, bdesc0 + soff + kk * b_kstep, p.idesc,
                     (kb > kb0 || kk > 0) ? 1u : 0u);
          }
          if constexpr (CG == 2) tc_commit2_both(&empty[s]);
          else tc_commit(&empty[s]);
          if (gk < 4) FM_MARK(28 + gk);
        }
        __syncwarp();
      }
      if (elect_one()) {
        if constexpr (CG == 2) tc_commit2_both(&tfull[acc]);
        else tc_commit(&tfull[acc]);
        FM_MARK(4);
      }
      __syncwarp();
    }
  } else if (warp >= 2) {
    // ===== epilogue: TMEM -> registers -> swizzled smem tile -> TMA store / reduce-add =====
    // Eight warps: warp w reads TMEM lane quarter w % 4 (32 rows, one row per thread);
    // the two warps of a quarter take alternate 32-column chunks, halving the per-warp
    // conversion / activation work (the epilogue is latency-bound at small tiles).  A
    // chunk is staged as a [32 rows][32 cols] box in smem with the TMA swizzle (128 B
    // rows for fp32, 64 B rows for bf16: conflict-free 16-byte st.shared) and written by
    // one TMA bulk store, or a TMA bulk reduce-add (fp32 grad accumulation C += acc, done
    // in L2).  EB 4 KB staging buffers per warp: with EB = 2 a chunk is staged while the
    // previous chunk's store still reads its buffer (write-bound, small-K GEMMs).
#ifdef FM_PROBE_OBS
    if (threadIdx.x == 65 && blockIdx.x == 0)  // observer: when each of the first stages lands
      for (int q = 0; q < p.nk && q < 8 && q < STAGES; ++q) {
        mbar_wait(&full[q], 0);
        g_probe[10 + (q < 6 ? q : 5)] = clock64();
      }
    __syncwarp();
#endif
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int r0 = quarter * 32;
    uint8_t* sb0 = epi_smem + (warp - 2) * EB * 4096;
    const bool f32out = g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32;
    int issued = 0;  // chunks this warp has stored (buffer issued % EB was used EB chunks ago)
    int it = 0;
    // stream-K partial of unit v (a unit stores at most one: its first stream-K segment,
    // when that is not the first segment of its tile); per CTA 128 x BN fp32 in the
    // epilogue's fragment order [quarter][32-column chunk][float4 j][lane], so a warp's
    // float4 store or load is 512 contiguous bytes
    auto part_ptr = [&](int v, int c0) {
      return reinterpret_cast<float4*>(g.splitk_ws + ((size_t)v * CG + crank) * (size_t)(TC_BM * BN)) +
             ((quarter * (BN / 32) + c0 / 32) * 8) * 32 + lane;
    };
    auto release_acc = [&](int acc) {  // TMEM reads of this accumulator are complete
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(mapa_u32(smem_u32(&tempty[acc]), 0));
        else mbar_arrive(&tempty[acc]);
      }
    };
    for (int64_t w = it_begin; seg_more(w); ++it) {
      int tile, kb0, kb1;
      seg_of(w, tile, kb0, kb1);
      w = seg_next(w, tile, kb0, kb1);
      const int n0 = (tile % ntn) * BN;
      const int m0 = ((tile / ntn) % ntm) * TC_BM * CG + (int)crank * TC_BM, b = tile / (ntn * ntm);
      const int acc = NACC == 2 ? (it & 1) : 0, use = NACC == 2 ? (it >> 1) : it;
      const uint32_t tmem_acc = tmem_base + acc * BN;
      const int row = m0 + r0 + lane;
      const bool row_ok = row < g.M;
      // the per-row bf16 operand of the epilogue (Z for dGELU, the residual) and the bias
      // are read one chunk ahead, the first chunk before the accumulator is ready, so
      // their load latency hides under the mainloop / the previous chunk
      const bf16* xrow = nullptr;
      if (!f32out && row_ok) {
        if (g.epi == EPI_DGELU || g.epi == EPI_MUL_AUX)
          xrow = reinterpret_cast<const bf16*>(g.aux) + (int64_t)b * g.sAux + (int64_t)row * g.ldaux;
        else if (g.epi == EPI_STORE && g.resid)
          xrow = reinterpret_cast<const bf16*>(g.resid) + (int64_t)b * g.sR + (int64_t)row * g.ldr;
      }
      const bf16* brow = (!f32out && g.bias) ? reinterpret_cast<const bf16*>(g.bias) + (int64_t)b * g.sBias : nullptr;
      uint4 pf[4], pb[4];
      auto prefetch = [&](int c) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const bool in = n0 + c + 8 * i < g.N;  // N % 8 == 0: a 16-byte group is all in or all out
          pf[i] = (xrow && in) ? *reinterpret_cast<const uint4*>(xrow + n0 + c + 8 * i) : make_uint4(0, 0, 0, 0);
          pb[i] = (brow && in) ? *reinterpret_cast<const uint4*>(brow + n0 + c + 8 * i) : make_uint4(0, 0, 0, 0);
        }
      };
      auto unpack = [](const uint4* q, float* out) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t w4[4] = {q[i].x, q[i].y, q[i].z, q[i].w};
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            out[8 * i + 2 * j] = __uint_as_float(w4[j] << 16);
            out[8 * i + 2 * j + 1] = __uint_as_float(w4[j] & 0xFFFF0000u);
          }
        }
      };
      prefetch(half * 32);
      if constexpr (CG == 2) mbar_wait_cl_sleep(&tfull[acc], use & 1);
      else mbar_wait_sleep(&tfull[acc], use & 1);
      if (threadIdx.x == 64) FM_MARK(5);
      tc_fence_after();
      // ---- stream-K fix-up of a cut tile.  Its first segment (the owner: the end of unit
      // uf's range, so the last work of that unit) keeps its accumulator in TMEM; every later
      // segment is the first stream-K work of its unit (uf+1 ..), stores its raw fp32
      // accumulator, frees TMEM at once and counts itself written.  The owner waits for the
      // count — those segments started before it and wait on nothing, so the wait cannot be
      // circular — and adds them to its own in segment order (a fixed order: deterministic).
      int uf = 0, nseg = 1;
      bool owner = false;
      if (sk && !(kb0 == 0 && kb1 == p.nk)) {
        const int64_t xr = (int64_t)tile * p.nk - sk_base;
        uf = (int)(((xr + 1) * nunits - 1) / sk_total);
        nseg = (int)(((xr + p.nk) * nunits - 1) / sk_total) - uf + 1;
        unsigned int* ctr = g.splitk_tick + (size_t)(tile - dp_tiles) * CG + crank;  // partials written
        if (unit != uf) {
#pragma unroll 1
          for (int c0 = half * 32; c0 < BN; c0 += 64) {
            if (n0 + c0 >= g.N) break;  // warp-uniform
            uint32_t r[32];
            tmem_ld32(tmem_acc + ((uint32_t)r0 << 16) + c0, r);
            float4* dst = part_ptr(unit, c0);
#pragma unroll
            for (int j = 0; j < 8; ++j)
              __stcg(dst + 32 * j, make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]),
                                               __uint_as_float(r[4 * j + 2]), __uint_as_float(r[4 * j + 3])));
          }
          release_acc(acc);
          __threadfence();  // the partial is visible before it is counted
          named_bar_sync(2, 256);
          if (threadIdx.x == 64) atomicAdd(ctr, 1u);
          continue;
        }
        owner = true;
        if (threadIdx.x == 64) {
          FM_HANG_DECL;
          while (true) {
            unsigned int v;
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
            if (v >= (unsigned int)(nseg - 1) || FM_HANG(tile, v)) break;
            __nanosleep(64);
          }
          *ctr = 0u;  // every later segment has written: ready for the next launch
        }
        named_bar_sync(2, 256);
        __threadfence();
      }
#pragma unroll 1
      for (int c0 = half * 32; c0 < BN; c0 += 64) {
        const int nb = n0 + c0;
        if (nb >= g.N) break;  // warp-uniform
        uint32_t r[32];
        tmem_ld32(tmem_acc + ((uint32_t)r0 << 16) + c0, r);
        for (int s2 = 1; owner && s2 < nseg; ++s2) {  // + the later segments, in order
          const float4* src = part_ptr(uf + s2, c0);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 q = __ldcg(src + 32 * j);
            r[4 * j] = __float_as_uint(__uint_as_float(r[4 * j]) + q.x);
            r[4 * j + 1] = __float_as_uint(__uint_as_float(r[4 * j + 1]) + q.y);
            r[4 * j + 2] = __float_as_uint(__uint_as_float(r[4 * j + 2]) + q.z);
            r[4 * j + 3] = __float_as_uint(__uint_as_float(r[4 * j + 3]) + q.w);
          }
        }
        if (threadIdx.x == 64 && c0 == 0) FM_MARK(9);
        float xv[32], bv[32];
        unpack(pf, xv);
        unpack(pb, bv);
        if (c0 + 64 < BN) prefetch(c0 + 64);
        float v[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * g.alpha + bv[i];  // bias 0 past N
        const int nvalid = min(32, g.N - nb);
        if (g.epi == EPI_STORE && g.resid && row_ok) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] += xv[i];  // zeros past N
        } else if (g.epi == EPI_DGELU && row_ok) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= (i < nvalid) ? gelu_grad_f(xv[i]) : 0.f;
        } else if (g.epi == EPI_MUL_AUX && row_ok) {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] *= xv[i];  // zeros past N
        }
        if (threadIdx.x == 64 && c0 == 0) FM_MARK(10);
        // the staging buffer is free once the store that used it EB chunks ago has read it
        uint8_t* sb = sb0 + (issued % EB) * 4096;
        if (issued >= EB) {
          if (lane == 0) bulk_wait_read<EB - 1>();
          __syncwarp();
        }
        if (threadIdx.x == 64 && c0 == 0) FM_MARK(11);
        if (f32out) {
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4 q = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            *reinterpret_cast<float4*>(sb + lane * 128 + ((j ^ (lane & 7)) << 4)) = q;
          }
        } else if (g.epi == EPI_BIAS_GELU_G) {
          // aux = GELU'(bf16(Z)), C = GELU(bf16(Z)): one erf and one exp per element
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            float hh[8], dd[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float z = __bfloat162float(__float2bfloat16_rn(v[8 * j + i]));
              const float cdf = 0.5f * (1.0f + erff(z * 0.70710678118654752f));
              hh[i] = z * cdf;
              dd[i] = cdf + z * __expf(-0.5f * z * z) * 0.39894228040143268f;
            }
            uint4 hq, dq;
            hq.x = pack_bf16x2(hh[0], hh[1]); hq.y = pack_bf16x2(hh[2], hh[3]);
            hq.z = pack_bf16x2(hh[4], hh[5]); hq.w = pack_bf16x2(hh[6], hh[7]);
            dq.x = pack_bf16x2(dd[0], dd[1]); dq.y = pack_bf16x2(dd[2], dd[3]);
            dq.z = pack_bf16x2(dd[4], dd[5]); dq.w = pack_bf16x2(dd[6], dd[7]);
            const int off = lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4);
            *reinterpret_cast<uint4*>(sb + off) = hq;
            *reinterpret_cast<uint4*>(sb + 2048 + off) = dq;
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
        if (threadIdx.x == 64 && c0 == 0) FM_MARK(12);
        fence_async_smem();
        __syncwarp();
        if (threadIdx.x == 64 && c0 == 0) FM_MARK(13);
        if (lane == 0) {
          if (g.epi == EPI_ACC_F32) {
            tma_reduce_add_3d(&tma_c, sb, nb, m0 + r0, b);
          } else if (g.epi == EPI_STORE_F32) {
            tma_store_3d(&tma_c, sb, nb, m0 + r0, b);
          } else {
            tma_store_3d(&tma_c, sb, nb, m0 + r0, b);
            if (g.epi == EPI_BIAS_GELU || g.epi == EPI_BIAS_GELU_G) tma_store_3d(&tma_aux, sb + 2048, nb, m0 + r0, b);
          }
          bulk_commit();
        }
        ++issued;
      }
      release_acc(acc);  // TMEM reads of this tile are complete
    }
    if (threadIdx.x == 64) FM_MARK(6);
    if (lane == 0) bulk_wait<0>();
    if (threadIdx.x == 64) FM_MARK(7);
    __syncwarp();
    tc_fence_before();
  }
  __syncthreads();
  if constexpr (CG == 2) {  // neither CTA leaves (or frees TMEM) while its peer may still signal it
    tc_fence_before();
    cluster_sync_all();
  }
  if (threadIdx.x == 0) FM_MARK(8);
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    if constexpr (CG == 2) tmem_dealloc2(tmem_base, tmem_cols);
    else tmem_dealloc(tmem_base, tmem_cols);
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

template <int BN, int STAGES, int EB = 1, int CG = 1, bool SK = false>
static int launch_tc(const GemmArgs& g, cudaStream_t s) {
  constexpr int streamk = SK ? 1 : 0;
  constexpr int BNL = BN / CG;
  CUtensorMap ma, mb;
  int rc;
  if (!g.a_mmajor) rc = make_map(&ma, g.A, g.K, g.M, g.batch, g.lda, g.sA, TC_BM);
  else rc = make_map(&ma, g.A, g.M, g.K, g.batch, g.lda, g.sA, TC_BK);
  if (rc) return rc;
  constexpr int NSUB = (CG == 2 && BN > 256) ? BN / 256 : 1;
  if (g.b_kmajor) rc = make_map(&mb, g.B, g.K, g.N, g.batch, g.ldb, g.sB, BNL / NSUB);
  else rc = make_map(&mb, g.B, g.N, g.K, g.batch, g.ldb, g.sB, TC_BK);
  if (rc) return rc;
  // output tiles: [32 rows][32 cols] boxes, fp32 (reduce-add, SW128) or bf16 (store, SW64)
  CUtensorMap mc, maux;
  const bool f32 = g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32;
  rc = make_map(&mc, g.C, g.N, g.M, g.batch, g.ldc, g.sC, 32, 32, f32,
                f32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B);
  if (rc) return rc;
  maux = mc;
  if (g.epi == EPI_BIAS_GELU || g.epi == EPI_BIAS_GELU_G) {
    rc = make_map(&maux, g.aux, g.N, g.M, g.batch, g.ldaux, g.sAux, 32, 32, false, CU_TENSOR_MAP_SWIZZLE_64B);
    if (rc) return rc;
  }
  TcArgs p;
  p.g = g;
  p.a_mmajor = g.a_mmajor;
  p.b_kmajor = g.b_kmajor;
  p.nk = (g.K + TC_BK - 1) / TC_BK;
  p.dbg = g_tc_debug;
  p.streamk = streamk;
  // kind::f16 instruction descriptor: D f32, A/B bf16, majors, N>>3, M>>4
  p.idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(g.a_mmajor ? 1 : 0) << 15) |
            ((uint32_t)(g.b_kmajor ? 0 : 1) << 16) | ((uint32_t)((BN / NSUB) >> 3) << 17) |
            ((uint32_t)((TC_BM * CG) >> 4) << 24);
  const size_t smem_max = (size_t)STAGES * (TC_BM * TC_BK * 2 + BNL * TC_BK * 2) + EB * 32768 + 1024 + 256;
  auto kern = gemm_tc_kernel<BN, STAGES, EB, CG, SK>;
  static bool attr_set = (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max), true);
  (void)attr_set;
  static int num_sms = 0;
  if (!num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev);
    if (num_sms <= 0) num_sms = 148;
  }
  const int64_t tiles = (int64_t)((g.N + BN - 1) / BN) * ((g.M + TC_BM * CG - 1) / (TC_BM * CG)) * g.batch;
  const int units = (g.max_sms > 0 && g.max_sms < num_sms ? g.max_sms : num_sms) / CG;
  const int nu = streamk ? units : (int)(tiles < units ? tiles : units);
  const size_t smem = (tiles <= nu && !streamk) ? smem_max - EB * 32768 : smem_max;
  if constexpr (CG == 2)
    launch_kc(kern, dim3(2 * nu), TC_THREADS, smem, s, dim3(2, 1, 1), ma, mb, mc, maux, p);
  else
    launch_k(kern, dim3(nu), TC_THREADS, smem, s, ma, mb, mc, maux, p);
  return (int)cudaGetLastError();
}

int gemm_tc(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0 || g.K <= 0) return 0;
  if (g_tc_debug & 1) return gemm_simt(g, DT_BF16, s);
  if (int rc = gemm_tc_init()) return rc;
  // Tile width (measured, tools/gemm_microbench.py): BN=256 (best MMA/operand efficiency)
  // whenever it still yields >= 48 tiles; small, latency-bound GEMMs get narrower tiles
  // and more CTAs.
  // stream-K needs the caller's scratch (one partial tile per CTA, one counter per cut tile
  // and CTA), a partial wave to balance, and at least 2 k-blocks of it per unit (no unit
  // may be left without stream-K work: the fix-up counts on one segment per unit)
  auto sk_ok = [&](int bn, int cg) {
    const int64_t units = 148 / cg, nk = (g.K + TC_BK - 1) / TC_BK;
    const int64_t t = (int64_t)((g.M + TC_BM * cg - 1) / (TC_BM * cg)) * g.batch * ((g.N + bn - 1) / bn);
    return g_force_sk != 1 && g.splitk_ws && g.splitk_ws_floats >= (size_t)units * cg * TC_BM * bn &&
           g.splitk_ticks >= (size_t)(units * cg) && (t % units) * nk >= 2 * units;
  };
  if (g_force_cg == 2) {
    if (g_force_bn == 128) return launch_tc<128, 8, 1, 2>(g, s);
    if (g_force_bn == 512) return launch_tc<512, 4, 1, 2>(g, s);
    return g_force_sk == 2 && sk_ok(256, 2) ? launch_tc<256, 6, 1, 2, true>(g, s) : launch_tc<256, 6, 1, 2>(g, s);
  }
  if (g_force_bn == 256) return g_force_sk == 2 && sk_ok(256, 1) ? launch_tc<256, 4, 1, 1, true>(g, s) : launch_tc<256, 4>(g, s);
  if (g_force_bn == 192) return launch_tc<192, 4>(g, s);
  if (g_force_bn == 128) return launch_tc<128, 6>(g, s);
  if (g_force_bn == 64) return launch_tc<64, 8>(g, s);
  const bool f32out = g.epi == EPI_ACC_F32 || g.epi == EPI_STORE_F32;
  const int64_t mt = (int64_t)((g.M + TC_BM - 1) / TC_BM) * g.batch;
  auto tiles = [&](int bn) { return mt * ((g.N + bn - 1) / bn); };
  // write-bound fp32 wgrads (K <= 256, many tiles: the c4 expert dW) on single CTAs take a
  // 3-stage ring and double-buffered epilogue staging (tools/probe/gemm_probe.cu: -2..-6%);
  // with more than 128 rows they go to the CTA pairs below (c4 dW1 1016 -> 957 us)
  if (g.N >= 256 && f32out && g.K <= 4 * TC_BK && tiles(256) >= 4 * 148 && (g.M <= TC_BM || g_force_cg == 1))
    return launch_tc<256, 3, 2>(g, s);
  if (g.N >= 256 && tiles(256) >= 48) {
    // Wave-quantised cost of the candidate tilings: waves x BN / eff, eff measured per SM at
    // the dsv2s / c3 / c4 shapes (tools/gemm_microbench.py, r02): CTA pairs on 256 x 256
    // tiles (cta_group::2, half the B operand per SM: the L2-bound mainloop) 1.0, one CTA
    // 128 x 256 0.89, one CTA 128 x 192 0.78.  192 columns only as a single wave: they fill
    // the SMs where 256 leave most of a wave idle (the T_r-row MHA projections: 80 -> 108 of
    // 148 SMs, 32 -> 28 us); with every SM busy the extra operand bytes per FLOP lose to the
    // pairs (dsv2s E1 73 vs 68 us), and so they do on long K (> 8192); measured on the
    // unbatched projections only, so the batched expert GEMMs keep 256.  The fp32 wgrads pair
    // too (dsv2s dW1, K = 512: 174 -> 136 us) since the epilogue's remote TMEM-release arrive
    // no longer carries a GPU-scope fence (tc_common.cuh mbar_arrive_cluster).
    auto cost = [](int64_t t, int slots, double w) { return (double)((t + slots - 1) / slots) * w; };
    const int64_t nk = (g.K + TC_BK - 1) / TC_BK;
    int pick = 1;
    double best = cost(tiles(256), 148, 256 / 0.89);
    const bool pairs_ok = g_force_cg == 0 && g.M > TC_BM;
    const int64_t mp = (int64_t)((g.M + 2 * TC_BM - 1) / (2 * TC_BM)) * g.batch;  // pair rows
    const int64_t t256 = mp * ((g.N + 255) / 256), t512 = mp * ((g.N + 511) / 512);
    if (pairs_ok) {
      const double c = cost(t256, 74, 256);
      if (c <= best) { best = c; pick = 2; }
    }
    if (g.batch == 1 && g.K <= 8192 && tiles(192) <= 148 && cost(tiles(192), 148, 192 / 0.78) < best) pick = 3;
    // 512-column pair tiles: two UMMAs per K-step share the A tile, 25% fewer L2->SMEM bytes
    // per FLOP — the bound once every SM is busy — where they need at most half the waves
    // of the 256-column pairs; not under the GELU epilogues (the single TMEM accumulator
    // leaves the activation unhidden).  dsv2s QKV 66.6 -> 64.4 us, expert dGELU 71.1 -> 66.4.
    if (pick == 2 && nk >= 32 && g.epi != EPI_BIAS_GELU && g.epi != EPI_BIAS_GELU_G &&
        2 * ((t512 + 73) / 74) <= (t256 + 73) / 74)
      pick = 5;
    // Stream-K on the 256-column pairs where the pairs are under one wave or K is long:
    // dsv2s dX (40 pair tiles, K = 15360) 79.4 -> 65.0 us, o-proj / dctx (K = 5120) 30.4 ->
    // 29.4 us.  Short K loses to the fix-up (E2, K = 1536: 58.6 -> 67.2 us).
    if (pairs_ok && sk_ok(256, 2) && (g_force_sk == 2 || (nk >= 64 && (t256 < 74 || nk >= 128)))) pick = 4;
    if (pick == 4) return launch_tc<256, 6, 1, 2, true>(g, s);
    if (pick == 5) return launch_tc<512, 4, 1, 2>(g, s);
    if (pick == 2) return launch_tc<256, 6, 1, 2>(g, s);
    if (pick == 3) return launch_tc<192, 4>(g, s);
    return launch_tc<256, 4>(g, s);
  }
  if (g.N >= 128 && tiles(128) >= 48) return launch_tc<128, 6>(g, s);
  return launch_tc<64, 8>(g, s);
}

}  // namespace fm
