// K6 on the 5th-generation tensor cores: flash attention forward and backward
// (S2 AT-attn and its backward in B5) for bf16, d_h in {64, 128}.
//
// Math per sequence s and head h (P:75 MHA; reading Q7: scale 1/sqrt(d_h), optional
// causal mask):  S = Q K^T * scale, P = softmax(S), ctx = P V, lse = log sum exp(S);
// backward: D = rowsum(dO ⊙ O), P = exp(S - lse), dP = dO V^T, dS = P ⊙ (dP - D),
// dV = P^T dO, dK = dS^T Q * scale, dQ = dS K * scale.
//
// Every product is a tcgen05.mma (cta_group::1, M = 128) with fp32 accumulators in
// TMEM; Q/K/V/dO tiles arrive by TMA (boxes {64 cols, 128 rows}, 128-byte swizzle);
// P, P^T and dS^T are written by the softmax warps straight into shared memory in
// the UMMA K-major swizzled layout and consumed as the A operand of the next MMA.
// The same smem tile of K (or V, Q, dO) serves as a K-major operand (contracting
// over d) and as an MN-major operand (contracting over rows), so no transposes.
//
// Warp roles (320 threads): warp 0 TMA producer, warp 1 TMEM owner + MMA issuer (one
// elected lane), warps 2..9 softmax / epilogue: one query (or key) row per thread, the
// two warps of a TMEM lane quarter splitting the tile's columns.
#include <cuda.h>
#include "common.cuh"
#include "kernels.h"
#include "tc_common.cuh"

namespace fm {

constexpr int AT_THREADS = 320;  // producer, MMA, 8 softmax warps (two per TMEM lane quarter)
constexpr float LOG2E = 1.4426950408889634f;
constexpr float LN2 = 0.6931471805599453f;

// Operand built from TMA boxes of {64 cols, 128 rows} (16 KB each, SW128):
// K-major (contract over the 64-col dim): k-step kk of 16 -> box kk/4, +32 B*(kk%4).
FM_DEV uint64_t kdesc(uint32_t base, int kk) {
  return umma_desc(base + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024);
}
// MN-major (contract over the 128 rows): k-step kk of 16 rows -> +2048 B; 64-col blocks 16 KB apart.
FM_DEV uint64_t mdesc(uint32_t base, int kk) { return umma_desc(base + kk * 2048, 16384, 1024); }
// The same as a base descriptor plus a constant added to its 14-bit address field, so
// the issuing loop only does 64-bit adds of uniform values.
FM_DEV uint64_t kdesc0(uint32_t base) { return umma_desc(base, 16, 1024); }
FM_DEV uint64_t mdesc0(uint32_t base) { return umma_desc(base, 16384, 1024); }
FM_DEV constexpr uint64_t kstep(int kk) { return (uint64_t)(((kk >> 2) * 16384 + (kk & 3) * 32) >> 4); }
FM_DEV constexpr uint64_t mstep(int kk) { return (uint64_t)((kk * 2048) >> 4); }

FM_DEV uint8_t* align1k(uint8_t* p) {
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(p) + 1023) & ~uintptr_t(1023));
}

// Write 32 fp32 values of row `row` (keys/queries c0..c0+31 of a 128-wide tile) as bf16
// into a K-major SW128 tile made of two {64, 128} boxes.
FM_DEV void st_row32_bf16(uint8_t* tile, int row, int c0, const float* v) {
  uint8_t* box = tile + (c0 >> 6) * 16384 + row * 128;
  const int cbase = (c0 & 63) >> 3;  // 16-byte chunk index of c0 within the 128-byte row
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    uint4 q;
    q.x = pack_bf16x2(v[8 * j], v[8 * j + 1]);
    q.y = pack_bf16x2(v[8 * j + 2], v[8 * j + 3]);
    q.z = pack_bf16x2(v[8 * j + 4], v[8 * j + 5]);
    q.w = pack_bf16x2(v[8 * j + 6], v[8 * j + 7]);
    *reinterpret_cast<uint4*>(box + (((cbase + j) ^ (row & 7)) << 4)) = q;
  }
}

FM_DEV void store_row_bf16(bf16* dst, const float* v, int n) {  // n multiple of 8
#pragma unroll
  for (int i = 0; i < 32; i += 8)
    if (i < n) store16<bf16>(dst + i, v + i);
}

// D = <O_row, dO_row> over one head's DH columns (16-byte loads)
template <int DH>
FM_DEV float row_dot_bf16(const bf16* o, const bf16* g) {
  float acc = 0.f;
#pragma unroll 4
  for (int c = 0; c < DH; c += 8) {
    float a[8], b[8];
    load16<bf16>(o + c, a);
    load16<bf16>(g + c, b);
#pragma unroll
    for (int i = 0; i < 8; ++i) acc = fmaf(a[i], b[i], acc);
  }
  return acc;
}

// Row ranges.  Sequences are N rows apart; a launch computes the "own" rows at positions
// [p0, p0 + np) of each sequence (queries for fwd / dQ, keys for dK/dV).  Whole-sequence
// chunks use p0 = 0, np = N; a token chunk (chunked prefill, causal only) is a slice of
// one sequence, attending to the keys before it.
// ============================================================== forward
// grid (ceil(np/128), H, n_seq); qkv map over rows [0, (n_seq-1)·N + p0 + np) so rows past
// the own range (not yet computed in a token chunk) load as zeros.
template <int DH>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_fwd_tc_kernel(const __grid_constant__ CUtensorMap tq, bf16* ctx, float* lse, int N, int p0, int np,
                       int M, int H, int causal, float scale_log2) {
  constexpr int NB = DH / 64;
  constexpr uint32_t TILE = 128 * DH * 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = align1k(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sK0 = smem + TILE;
  uint8_t* sV0 = smem + 2 * TILE;
  uint8_t* sK1 = smem + 3 * TILE;
  uint8_t* sV1 = smem + 4 * TILE;
  uint8_t* sP = smem + 5 * TILE;  // 32 KB: [2 boxes][128 q][64 keys]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 32768);
  uint64_t* bar_q = bars;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* p_full = bars + 7;
  uint64_t* o_done = bars + 8;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 9);
  float* xch = reinterpret_cast<float*>(bars + 16);  // [3][2 halves][128 rows]: row max (tile parity), row sum

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // longest-first: linear block L -> query tile nt-1-L/(n_seq·H) (causal work grows with qt)
  const int per = gridDim.y * gridDim.z;
  const int L = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  const int lv = L / per, r = L - lv * per;
  const int qt = gridDim.x - 1 - lv, h = r % gridDim.y, sq = r / gridDim.y;
  const int q0 = p0 + qt * 128, row_base = sq * N;  // q0: position of the tile's first query
  int nkv = (N + 127) / 128;
  if (causal) nkv = min(nkv, (min(p0 + np, q0 + 128) + 127) / 128);

  if (warp == 0 && lane == 0) {
    mbar_init(bar_q, 1);
    for (int i = 0; i < 2; ++i) { mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1); mbar_init(&s_full[i], 1); }
    mbar_init(p_full, 256);
    mbar_init(o_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tq)) : "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  FM_PDL_ENTRY();
  const uint32_t tO = tmem + 256;

  if (warp == 0) {
    // producer: whole warp walks the K/V ring, one elected lane issues the TMA loads
    if (elect_one()) {
      mbar_expect_tx(bar_q, TILE);
      for (int i = 0; i < NB; ++i) tma_load_2d(sQ + i * 16384, &tq, bar_q, h * DH + 64 * i, row_base + q0);
    }
    __syncwarp();
    for (int j = 0; j < nkv; ++j) {
      const int st = j & 1;
      if (j >= 2) mbar_wait_sleep(&kv_empty[st], ((j >> 1) - 1) & 1);
      uint8_t* sK = st ? sK1 : sK0;
      uint8_t* sV = st ? sV1 : sV0;
      if (elect_one()) {
        mbar_expect_tx(&kv_full[st], 2 * TILE);
        for (int i = 0; i < NB; ++i) {
          tma_load_2d(sK + i * 16384, &tq, &kv_full[st], M + h * DH + 64 * i, row_base + j * 128);
          tma_load_2d(sV + i * 16384, &tq, &kv_full[st], 2 * M + h * DH + 64 * i, row_base + j * 128);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    // MMA issuer: whole warp waits, one elected lane issues
    constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);  // Q (K-major) x K^T (K-major)
    constexpr uint32_t id_o = idesc_bf16(128, DH, 0, 1);   // P (K-major) x V (MN-major)
    const uint64_t dQ = kdesc0(smem_u32(sQ)), dP = kdesc0(smem_u32(sP));
    const uint64_t dK0 = kdesc0(smem_u32(sK0)), dK1 = kdesc0(smem_u32(sK1));
    const uint64_t dV0 = mdesc0(smem_u32(sV0)), dV1 = mdesc0(smem_u32(sV1));
    mbar_wait(bar_q, 0);
    auto issue_s = [&](int j) {
      const int st = j & 1;
      mbar_wait(&kv_full[st], (j >> 1) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc_mma(tmem + st * 128, dQ + kstep(kk), (st ? dK1 : dK0) + kstep(kk), id_s, kk > 0);
        tc_commit(&s_full[st]);
      }
      __syncwarp();
    };
    issue_s(0);
    for (int j = 0; j < nkv; ++j) {
      if (j + 1 < nkv) issue_s(j + 1);
      mbar_wait_sleep(p_full, j & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc_mma(tO, dP + kstep(kk), ((j & 1) ? dV1 : dV0) + mstep(kk), id_o, (j > 0 || kk > 0));
        tc_commit(o_done);
        tc_commit(&kv_empty[j & 1]);
      }
      __syncwarp();
    }
  } else {
    // ===== softmax warps: thread = query row; the two warps of a TMEM lane quarter take
    // key columns [64·half, 64·half + 64) of each S tile and O columns [DH/2·half, ..).
    // They share the running row max through shared memory (one 64-thread named
    // barrier per tile); the row sums stay per half until the end.
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int rloc = quarter * 32 + lane;
    const int qrow = q0 + rloc;                      // position in the sequence
    const bool own = qt * 128 + rloc < np;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    constexpr int OC = DH / 64;                      // O chunks of 32 columns per half
    float m = -INFINITY, l = 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(&s_full[j & 1], (j >> 1) & 1);
      tc_fence_after();
      const uint32_t tS = tmem + lane_off + (j & 1) * 128;
      float mx = -INFINITY;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = 2 * half + cc;
        uint32_t r[32];
        tmem_ld32(tS + c * 32, r);
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int key = j * 128 + c * 32 + i;
          const bool ok = key < N && (!causal || key <= qrow);
          if (ok) mx = fmaxf(mx, __uint_as_float(r[i]) * scale_log2);
        }
      }
      float* xm = xch + (j & 1) * 256;  // double-buffered: the partner read the other one a tile ago
      xm[half * 128 + rloc] = mx;
      named_bar_sync(2 + quarter, 64);
      mx = fmaxf(mx, xm[(half ^ 1) * 128 + rloc]);
      const float m_new = fmaxf(m, mx);
      const float corr = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
      const float msub = (m_new == -INFINITY) ? 0.f : m_new;
      if (j > 0) {
        mbar_wait(o_done, (j - 1) & 1);  // PV_{j-1} done: O is stable and P smem is free
        tc_fence_after();
        if (__any_sync(0xffffffffu, corr != 1.f)) {
#pragma unroll 1
          for (int cc = 0; cc < OC; ++cc) {
            const int c = half * OC + cc;
            uint32_t r[32];
            tmem_ld32(tO + lane_off + c * 32, r);
#pragma unroll
            for (int i = 0; i < 32; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * corr);
            tmem_st32(tO + lane_off + c * 32, r);
          }
        }
      }
      float rs = 0.f;
#pragma unroll
      for (int cc = 0; cc < 2; ++cc) {
        const int c = 2 * half + cc;
        uint32_t r[32];
        tmem_ld32(tS + c * 32, r);
        float p[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int key = j * 128 + c * 32 + i;
          const bool ok = key < N && (!causal || key <= qrow);
          p[i] = ok ? exp2f(__uint_as_float(r[i]) * scale_log2 - msub) : 0.f;
          rs += p[i];
        }
        st_row32_bf16(sP, rloc, c * 32, p);
      }
      l = l * corr + rs;
      m = m_new;
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(o_done, (nkv - 1) & 1);
    tc_fence_after();
    xch[512 + half * 128 + rloc] = l;
    named_bar_sync(2 + quarter, 64);
    l += xch[512 + (half ^ 1) * 128 + rloc];
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* dst = ctx + (int64_t)(row_base + qrow) * M + h * DH;
#pragma unroll 1
    for (int cc = 0; cc < OC; ++cc) {
      const int c = half * OC + cc;
      uint32_t r[32];
      tmem_ld32(tO + lane_off + c * 32, r);
      float v[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * inv;
      if (own) store_row_bf16(dst + c * 32, v, 32);
    }
    if (own && half == 0) lse[(int64_t)(row_base + qrow) * H + h] = (m + log2f(l)) * LN2;
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================== backward: dK, dV
// Q/dO tiles of the dK/dV half in flight: two for d_h = 64 (the next tile loads under the
// current one), one for d_h = 128 (shared memory).
template <int DH>
constexpr int DKDV_QSTAGES = DH == 64 ? 2 : 1;

// grid (ceil(np/128) own key tiles, H, n_seq); query tiles of 128 rows from the key tile's
// first row (causal) to N.  TMEM: S^T [0,128), dP^T [128,256), dV, dK.
template <int DH>
__device__ __forceinline__ void attn_bwd_dkdv_body(const CUtensorMap& tq, const CUtensorMap& tdo, const float* lse,
                                                   const bf16* ctxO, const bf16* dctx, bf16* dqkv, int N, int p0,
                                                   int np, int M, int H, int causal, float scale_log2, float scale,
                                                   uint8_t* smem_raw, int kt, int h, int sq) {
  constexpr int NB = DH / 64;
  constexpr uint32_t TILE = 128 * DH * 2;
  constexpr int QST = DKDV_QSTAGES<DH>;  // Q/dO tiles in flight (the next one loads under this one)
  uint8_t* smem = align1k(smem_raw);
  uint8_t* sK = smem;
  uint8_t* sV = smem + TILE;
  uint8_t* sQ0 = smem + 2 * TILE;       // [QST] x {Q, dO}
  uint8_t* sP = smem + (2 + 2 * QST) * TILE;  // P^T  [keys][queries], 32 KB
  uint8_t* sdS = sP + 32768;          // dS^T [keys][queries], 32 KB
  float* sL = reinterpret_cast<float*>(sdS + 32768);  // lse (log2 units) of the q tile
  float* sD = sL + 128;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sD + 128);
  uint64_t* kv_bar = bars;
  uint64_t* q_full = bars + 1;         // [QST]
  uint64_t* q_empty = bars + 1 + QST;  // [QST]
  uint64_t* s_full = bars + 1 + 2 * QST;
  uint64_t* p_full = s_full + 1;
  uint64_t* mm_done = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = p0 + kt * 128, row_base = sq * N;
  // query tiles from the key tile's first row (causal) to N.  A token chunk's keys start
  // mid-sequence (p0 not a multiple of 128): a 128-aligned first tile would also load the
  // dO rows of EARLIER chunks, which this backward has not produced yet (stale or
  // uninitialised memory: 0·NaN = NaN through P = 0 and dS = 0); tiles starting at k0 read
  // only queries >= k0.  Whole-sequence chunks (p0 = 0) keep the 128-aligned tiles.
  const int qs0 = causal ? k0 : 0;
  const int niter = (N - qs0 + 127) / 128;

  if (warp == 0 && lane == 0) {
    mbar_init(kv_bar, 1);
    for (int i = 0; i < QST; ++i) { mbar_init(&q_full[i], 1); mbar_init(&q_empty[i], 1); }
    mbar_init(s_full, 1);
    mbar_init(p_full, 256);
    mbar_init(mm_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  FM_PDL_ENTRY();
  const uint32_t tST = tmem, tdPT = tmem + 128, tdV = tmem + 256, tdK = tmem + 256 + DH;

  if (warp == 0) {
    if (elect_one()) {
      mbar_expect_tx(kv_bar, 2 * TILE);
      for (int i = 0; i < NB; ++i) {
        tma_load_2d(sK + i * 16384, &tq, kv_bar, M + h * DH + 64 * i, row_base + k0);
        tma_load_2d(sV + i * 16384, &tq, kv_bar, 2 * M + h * DH + 64 * i, row_base + k0);
      }
    }
    __syncwarp();
    for (int it = 0; it < niter; ++it) {
      const int qr = row_base + qs0 + it * 128;
      const int st = it % QST;
      if (it >= QST) mbar_wait_sleep(&q_empty[st], ((it / QST) - 1) & 1);
      uint8_t* sQ = sQ0 + st * 2 * TILE;
      uint8_t* sdO = sQ + TILE;
      if (elect_one()) {
        mbar_expect_tx(&q_full[st], 2 * TILE);
        for (int i = 0; i < NB; ++i) {
          tma_load_2d(sQ + i * 16384, &tq, &q_full[st], h * DH + 64 * i, qr);
          tma_load_2d(sdO + i * 16384, &tdo, &q_full[st], h * DH + 64 * i, qr);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t id_g = idesc_bf16(128, DH, 0, 1);
    const uint64_t dK = kdesc0(smem_u32(sK)), dV = kdesc0(smem_u32(sV)), dP = kdesc0(smem_u32(sP)),
                   dS = kdesc0(smem_u32(sdS));
    const uint64_t dQk0 = kdesc0(smem_u32(sQ0)), dQm0 = mdesc0(smem_u32(sQ0));
    mbar_wait(kv_bar, 0);
    for (int it = 0; it < niter; ++it) {
      const int st = it % QST;
      const uint64_t qoff = (uint64_t)((uint32_t)(st * 2 * TILE) >> 4), ooff = qoff + (TILE >> 4);
      const uint64_t dQk = dQk0 + qoff, dOk = dQk0 + ooff, dQm = dQm0 + qoff, dOm = dQm0 + ooff;
      mbar_wait(&q_full[st], (it / QST) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc_mma(tST, dK + kstep(kk), dQk + kstep(kk), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc_mma(tdPT, dV + kstep(kk), dOk + kstep(kk), id_s, kk > 0);
        tc_commit(s_full);
      }
      __syncwarp();
      mbar_wait_sleep(p_full, it & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc_mma(tdV, dP + kstep(kk), dOm + mstep(kk), id_g, (it > 0 || kk > 0));
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc_mma(tdK, dS + kstep(kk), dQm + mstep(kk), id_g, (it > 0 || kk > 0));
        tc_commit(&q_empty[st]);
        tc_commit(mm_done);
      }
      __syncwarp();
    }
  } else {
    // ===== thread = key row; the two warps of a TMEM lane quarter take query columns
    // [64·half, 64·half + 64) of each tile and dV/dK columns [DH/2·half, ..)
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int kloc = quarter * 32 + lane;
    const int key = k0 + kloc;
    const int kend = p0 + np;  // own keys: key < kend
    const bool own = key < kend;
    const int t256 = threadIdx.x - 64;  // 0..255
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int it = 0; it < niter; ++it) {
      const int qbase = qs0 + it * 128;
      named_bar_sync(1, 256);  // everyone is done reading sL/sD of the previous tile
      if (t256 < 128) {
        const int qi = qbase + t256;
        sL[t256] = qi < N ? lse[(int64_t)(row_base + qi) * H + h] * LOG2E : 0.f;
      } else {
        const int qi = qbase + t256 - 128;
        const int64_t ro = (int64_t)(row_base + qi) * M + h * DH;
        sD[t256 - 128] = qi < N ? row_dot_bf16<DH>(ctxO + ro, dctx + ro) : 0.f;
      }
      named_bar_sync(1, 256);
      mbar_wait(s_full, it & 1);
      tc_fence_after();
      if (it > 0) {
        mbar_wait(mm_done, (it - 1) & 1);  // previous dV/dK MMAs finished reading P^T, dS^T
        tc_fence_after();
      }
#pragma unroll 1
      for (int c = 2 * half; c < 2 * half + 2; ++c) {
        uint32_t rs[32], rp[32];
        tmem_ld32(tST + lane_off + c * 32, rs);
        tmem_ld32(tdPT + lane_off + c * 32, rp);
        float p[32], ds[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int ql = c * 32 + i;
          const int qi = qbase + ql;
          const bool ok = qi < N && key < kend && (!causal || key <= qi);
          const float pv = ok ? exp2f(__uint_as_float(rs[i]) * scale_log2 - sL[ql]) : 0.f;
          p[i] = pv;
          ds[i] = pv * (__uint_as_float(rp[i]) - sD[ql]);  // rows past N / own range: finite, pv = 0
        }
        st_row32_bf16(sP, kloc, c * 32, p);
        st_row32_bf16(sdS, kloc, c * 32, ds);
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(mm_done, (niter - 1) & 1);
    tc_fence_after();
    bf16* row = dqkv + (int64_t)(row_base + key) * 3 * M;
#pragma unroll 1
    for (int c = half * (DH / 64); c < (half + 1) * (DH / 64); ++c) {
      uint32_t r[32];
      float v[32];
      tmem_ld32(tdV + lane_off + c * 32, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = niter > 0 ? __uint_as_float(r[i]) : 0.f;
      if (own) store_row_bf16(row + 2 * M + h * DH + c * 32, v, 32);
      tmem_ld32(tdK + lane_off + c * 32, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = niter > 0 ? __uint_as_float(r[i]) * scale : 0.f;
      if (own) store_row_bf16(row + M + h * DH + c * 32, v, 32);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// ============================================================== backward: dQ
// grid (ceil(np/128) own query tiles, H, n_seq).  TMEM: S [0,128), dP [128,256), dQ [256, 256+DH).
template <int DH, int STAGES>
__device__ __forceinline__ void attn_bwd_dq_body(const CUtensorMap& tq, const CUtensorMap& tdo, const float* lse,
                                                 const bf16* ctxO, const bf16* dctx, bf16* dqkv, int N, int p0,
                                                 int np, int M, int H, int causal, float scale_log2, float scale,
                                                 uint8_t* smem_raw, int qt, int h, int sq) {
  constexpr int NB = DH / 64;
  constexpr uint32_t TILE = 128 * DH * 2;
  uint8_t* smem = align1k(smem_raw);
  uint8_t* sQ = smem;
  uint8_t* sdO = smem + TILE;
  uint8_t* sKV = smem + 2 * TILE;                  // STAGES x {K, V}
  uint8_t* sdS = smem + (2 + 2 * STAGES) * TILE;   // 32 KB
  uint64_t* bars = reinterpret_cast<uint64_t*>(sdS + 32768);
  uint64_t* q_bar = bars;
  uint64_t* kv_full = bars + 1;            // [STAGES]
  uint64_t* kv_empty = bars + 1 + STAGES;  // [STAGES]
  uint64_t* s_full = bars + 1 + 2 * STAGES;
  uint64_t* p_full = s_full + 1;
  uint64_t* mm_done = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_full + 3);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int q0 = p0 + qt * 128, row_base = sq * N;
  int nkv = (N + 127) / 128;
  if (causal) nkv = min(nkv, (min(p0 + np, q0 + 128) + 127) / 128);

  if (warp == 0 && lane == 0) {
    mbar_init(q_bar, 1);
    for (int i = 0; i < STAGES; ++i) { mbar_init(&kv_full[i], 1); mbar_init(&kv_empty[i], 1); }
    mbar_init(s_full, 1);
    mbar_init(p_full, 256);
    mbar_init(mm_done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  FM_PDL_ENTRY();
  const uint32_t tS = tmem, tdP = tmem + 128, tdQ = tmem + 256;

  if (warp == 0) {
    if (elect_one()) {
      mbar_expect_tx(q_bar, 2 * TILE);
      for (int i = 0; i < NB; ++i) {
        tma_load_2d(sQ + i * 16384, &tq, q_bar, h * DH + 64 * i, row_base + q0);
        tma_load_2d(sdO + i * 16384, &tdo, q_bar, h * DH + 64 * i, row_base + q0);
      }
    }
    __syncwarp();
    for (int j = 0; j < nkv; ++j) {
      const int st = j % STAGES;
      if (j >= STAGES) mbar_wait_sleep(&kv_empty[st], ((j / STAGES) - 1) & 1);
      uint8_t* sK = sKV + st * 2 * TILE;
      uint8_t* sV = sK + TILE;
      if (elect_one()) {
        mbar_expect_tx(&kv_full[st], 2 * TILE);
        for (int i = 0; i < NB; ++i) {
          tma_load_2d(sK + i * 16384, &tq, &kv_full[st], M + h * DH + 64 * i, row_base + j * 128);
          tma_load_2d(sV + i * 16384, &tq, &kv_full[st], 2 * M + h * DH + 64 * i, row_base + j * 128);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {
    constexpr uint32_t id_s = idesc_bf16(128, 128, 0, 0);
    constexpr uint32_t id_g = idesc_bf16(128, DH, 0, 1);
    const uint64_t dQ = kdesc0(smem_u32(sQ)), dO = kdesc0(smem_u32(sdO)), dS = kdesc0(smem_u32(sdS));
    const uint64_t dKV0 = kdesc0(smem_u32(sKV)), mKV0 = mdesc0(smem_u32(sKV));
    mbar_wait(q_bar, 0);
    for (int j = 0; j < nkv; ++j) {
      const int st = j % STAGES;
      mbar_wait(&kv_full[st], (j / STAGES) & 1);
      tc_fence_after();
      const uint64_t soff = (uint64_t)((uint32_t)(st * 2 * TILE) >> 4), voff = (uint64_t)(TILE >> 4);
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc_mma(tS, dQ + kstep(kk), dKV0 + soff + kstep(kk), id_s, kk > 0);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) tc_mma(tdP, dO + kstep(kk), dKV0 + soff + voff + kstep(kk), id_s, kk > 0);
        tc_commit(s_full);
      }
      __syncwarp();
      mbar_wait_sleep(p_full, j & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) tc_mma(tdQ, dS + kstep(kk), mKV0 + soff + mstep(kk), id_g, (j > 0 || kk > 0));
        tc_commit(&kv_empty[st]);
        tc_commit(mm_done);
      }
      __syncwarp();
    }
  } else {
    // ===== thread = query row; the two warps of a TMEM lane quarter take key columns
    // [64·half, 64·half + 64) of each tile and dQ columns [DH/2·half, ..)
    const int quarter = warp & 3, half = (warp - 2) >> 2;
    const int rloc = quarter * 32 + lane;
    const int qrow = q0 + rloc;
    const int qend = p0 + np;  // own queries: qrow < qend
    const bool own = qrow < qend;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float L2 = own ? lse[(int64_t)(row_base + qrow) * H + h] * LOG2E : 0.f;
    const float Dq = own ? row_dot_bf16<DH>(ctxO + (int64_t)(row_base + qrow) * M + h * DH,
                                            dctx + (int64_t)(row_base + qrow) * M + h * DH) : 0.f;
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(s_full, j & 1);
      tc_fence_after();
      if (j > 0) {
        mbar_wait(mm_done, (j - 1) & 1);
        tc_fence_after();
      }
#pragma unroll 1
      for (int c = 2 * half; c < 2 * half + 2; ++c) {
        uint32_t rs[32], rp[32];
        tmem_ld32(tS + lane_off + c * 32, rs);
        tmem_ld32(tdP + lane_off + c * 32, rp);
        float ds[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int kj = j * 128 + c * 32 + i;
          const bool ok = qrow < qend && kj < N && (!causal || kj <= qrow);
          const float pv = ok ? exp2f(__uint_as_float(rs[i]) * scale_log2 - L2) : 0.f;
          ds[i] = pv * (__uint_as_float(rp[i]) - Dq);
        }
        st_row32_bf16(sdS, rloc, c * 32, ds);
      }
      fence_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
    }
    mbar_wait(mm_done, (nkv - 1) & 1);
    tc_fence_after();
    bf16* row = dqkv + (int64_t)(row_base + qrow) * 3 * M + h * DH;
#pragma unroll 1
    for (int c = half * (DH / 64); c < (half + 1) * (DH / 64); ++c) {
      uint32_t r[32];
      float v[32];
      tmem_ld32(tdQ + lane_off + c * 32, r);
#pragma unroll
      for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]) * scale;
      if (own) store_row_bf16(row + c * 32, v, 32);
    }
    tc_fence_before();
  }
  __syncthreads();
  if (warp == 1) {
    __syncwarp();
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

// dK/dV and dQ of one (sequence, head) run as one launch of grid (own tiles, H, 2·n_seq):
// each CTA takes one (role, sequence, head, tile) item (role 0: dK/dV of an own key
// tile, 1: dQ of an own query tile).  The two roles are independent (disjoint outputs, shared read-only inputs), so they co-run.
template <int DH, int STAGES>
__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_bwd_tc_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tdo,
                       const float* lse, const bf16* ctxO, const bf16* dctx, bf16* dqkv, int N, int p0, int np,
                       int M, int H, int causal, float scale_log2, float scale) {
  extern __shared__ uint8_t smem_raw[];
  // Longest-first order: CTAs are dispatched in linear block order, and a causal tile's
  // work grows with its distance from the diagonal end (dK/dV of key tile t: nt - t query
  // tiles; dQ of query tile t: t + 1 key tiles), so linear index L takes level
  // lv = L / (2·n_seq·H) = dK/dV tile lv and dQ tile nt-1-lv of every (sequence, head).
  // With more CTAs than SMs the heavy tiles start in the first wave.
  const int nt = gridDim.x, per = gridDim.y * gridDim.z;
  const int L = blockIdx.x + nt * (blockIdx.y + gridDim.y * blockIdx.z);
  const int lv = L / per, r = L - lv * per, rest = r >> 1;
  const int h = rest % gridDim.y, sq = rest / gridDim.y;
#ifdef FM_ATTN_LINEAR  // probe A/B only: the natural (tile, head, 2·seq + role) order
  if (blockIdx.z & 1)
    attn_bwd_dq_body<DH, STAGES>(tq, tdo, lse, ctxO, dctx, dqkv, N, p0, np, M, H, causal, scale_log2, scale,
                                 smem_raw, blockIdx.x, blockIdx.y, blockIdx.z >> 1);
  else
    attn_bwd_dkdv_body<DH>(tq, tdo, lse, ctxO, dctx, dqkv, N, p0, np, M, H, causal, scale_log2, scale, smem_raw,
                           blockIdx.x, blockIdx.y, blockIdx.z >> 1);
  return;
#endif
  if (r & 1)
    attn_bwd_dq_body<DH, STAGES>(tq, tdo, lse, ctxO, dctx, dqkv, N, p0, np, M, H, causal, scale_log2, scale,
                                 smem_raw, nt - 1 - lv, h, sq);
  else
    attn_bwd_dkdv_body<DH>(tq, tdo, lse, ctxO, dctx, dqkv, N, p0, np, M, H, causal, scale_log2, scale, smem_raw,
                           lv, h, sq);
}

// D[t][h] = sum_d dO[t][h*dh+d] * O[t][h*dh+d]: one warp per token, 16-byte loads;
// lane groups of dh/8 lanes reduce one head each (segmented shuffle reduction).
__global__ void attn_bwd_pre_tc_kernel(const bf16* ctx, const bf16* dctx, float* D, int T_, int M,
                                       int H) {
  FM_PDL_ENTRY();
  const int t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T_) return;
  const int dh = M / H, G = dh / 8;  // lanes per head (8 or 16)
  const bf16* o = ctx + (int64_t)t * M;
  const bf16* g = dctx + (int64_t)t * M;
  for (int m0 = lane * 8; m0 - lane * 8 < M; m0 += 256) {
    float acc = 0.f;
    if (m0 < M) {
      float a[8], b[8];
      load16<bf16>(o + m0, a);
      load16<bf16>(g + m0, b);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fmaf(a[i], b[i], acc);
    }
    for (int off = 1; off < G; off <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
    if (m0 < M && (lane % G) == 0) D[(int64_t)t * H + m0 / dh] = acc;
  }
}

// ------------------------------------------------------------ host
template <int DH>
static size_t fwd_smem() { return 5 * 128 * DH * 2 + 32768 + 1024 + 128 + 3072 + 256; }
template <int DH>
static size_t dkdv_smem() { return (2 + 2 * DKDV_QSTAGES<DH>) * 128 * DH * 2 + 65536 + 1024 + 1024 + 256; }
template <int DH, int ST>
static size_t dq_smem() { return (2 + 2 * ST) * 128 * DH * 2 + 32768 + 1024 + 256; }

template <int DH>
static int attn_fwd_tc_t(const void* qkv, void* ctx, float* lse, int nseq, int N, int p0, int np, int M, int H,
                         int causal, cudaStream_t s) {
  CUtensorMap tq;
  if (int rc = make_tmap_2d_bf16(&tq, qkv, 3 * M, (nseq - 1) * N + p0 + np, 3 * M, 64, 128)) return rc;
  auto k = attn_fwd_tc_kernel<DH>;
  const size_t smem = fwd_smem<DH>();
  static bool once = (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), true);
  (void)once;
  dim3 grid((np + 127) / 128, H, nseq);
  launch_k(k, grid, AT_THREADS, smem, s, tq, (bf16*)ctx, lse, N, p0, np, M, H, causal, LOG2E / sqrtf((float)DH));
  return (int)cudaGetLastError();
}

template <int DH>
static int attn_bwd_tc_t(const void* qkv, const void* ctx, const float* lse, const void* dctx, void* dqkv,
                         float* D, int nseq, int N, int p0, int np, int M, int H, int causal, cudaStream_t s) {
  CUtensorMap tq, tdo;
  if (int rc = make_tmap_2d_bf16(&tq, qkv, 3 * M, nseq * N, 3 * M, 64, 128)) return rc;
  if (int rc = make_tmap_2d_bf16(&tdo, dctx, M, nseq * N, M, 64, 128)) return rc;
  (void)D;  // D = rowsum(dO ⊙ O) is computed inside the two kernels
  const float scale = 1.0f / sqrtf((float)DH), sl2 = LOG2E * scale;
  constexpr int ST = DH == 128 ? 1 : 2;
  auto k = attn_bwd_tc_kernel<DH, ST>;
  const size_t sm = dkdv_smem<DH>() > dq_smem<DH, ST>() ? dkdv_smem<DH>() : dq_smem<DH, ST>();
  static bool once = (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm), true);
  (void)once;
  launch_k(k, dim3((np + 127) / 128, H, 2 * nseq), AT_THREADS, sm, s, tq, tdo, lse, (const bf16*)ctx,
           (const bf16*)dctx, (bf16*)dqkv, N, p0, np, M, H, causal, sl2, scale);
  return (int)cudaGetLastError();
}

bool attn_tc_supported(int dtype, int M, int H) {
  const int dh = M / H;
  return dtype == DT_BF16 && (dh == 64 || dh == 128) && !(attn_tc_debug_off());
}

int attn_fwd_tc(const void* qkv, void* ctx, float* lse, int nseq, int N, int p0, int np, int M, int H,
                int causal, cudaStream_t s) {
  if (M / H == 64) return attn_fwd_tc_t<64>(qkv, ctx, lse, nseq, N, p0, np, M, H, causal, s);
  return attn_fwd_tc_t<128>(qkv, ctx, lse, nseq, N, p0, np, M, H, causal, s);
}

int attn_bwd_tc(const void* qkv, const void* ctx, const float* lse, const void* dctx, void* dqkv, float* D,
                int nseq, int N, int p0, int np, int M, int H, int causal, cudaStream_t s) {
  if (M / H == 64) return attn_bwd_tc_t<64>(qkv, ctx, lse, dctx, dqkv, D, nseq, N, p0, np, M, H, causal, s);
  return attn_bwd_tc_t<128>(qkv, ctx, lse, dctx, dqkv, D, nseq, N, p0, np, M, H, causal, s);
}

}  // namespace fm
