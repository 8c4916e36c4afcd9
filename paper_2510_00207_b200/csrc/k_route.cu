// Gating, routing and token movement kernels of the FlowMoE block.
//   K1 gate_topk        (S4: logits = I'·Wg, softmax, top-k)
//   K2 route_scan       (S5: capacity positions C = ceil(f·k·B·N/E))
//   K3 permute_pack     (S5: rows -> A2A send buffer G(I') ∈ R^{E×C×M})
//   K7 unpermute_combine(S9: out[t] = Σ_j w_tj·Y[e_tj][pos_tj] (+I'))
//   K8 combine_bwd_pack (B1: dY = w·dO, dw = <dO, Y>)
//   K9 gather_gate_bwd  (B4: dI' = Σ dX + dlogits·Wgᵀ (+dO))
//   gate_wgrad          (B4: dWg += I'ᵀ·dlogits, deterministic split-T)
//   colsum_acc          (B2: db1, db2)
// All HBM-bound: 16-byte vector accesses, register tiles for the two small
// contractions with Wg (E <= 64 columns), deterministic reductions throughout.
// Readings: Q3 slot-major-then-token positions, Q4 top-k on fp32
// logits with ties -> lower index, Q5 renormalised top-k weights (k>=2) or raw
// softmax prob (k=1), Q6 no gate bias.
#include <cooperative_groups.h>
#include "common.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace fm {

// Phase probe (tools/probe/gate_probe.cu builds this file with -DFM_PROBE): clock64
// stamps of the gate kernel's phases in CTA 0 (slots 0-7) and in the scanning CTA (8-15).
#ifdef FM_PROBE
__device__ long long g_gprobe[24];
#define FM_GMARK(i) do { if (threadIdx.x == 0) g_gprobe[i] = clock64(); } while (0)
#else
#define FM_GMARK(i) do {} while (0)
#endif

FM_DEV uint32_t rt_smem(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// shared::cta address -> the same offset in cluster CTA `rank`'s shared memory
FM_DEV uint32_t rt_mapa(uint32_t a, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}

__device__ void route_scan_body(const int32_t* idx, int32_t* pos, int32_t* counts, int32_t* src, int T_,
                                int E, int k, int C, int* hist, int* warp_tot);

// ------------------------------------------------------------------ K1
// logits = A·Wg is a [T_r × M]·[M × E] product with E ≤ 64: HBM-bound on A.  A CTA
// covers TB tokens and one slice of M; each lane keeps a 4-token × EG-expert register
// tile (one 16-byte load of A per token feeds 4·EG·V FMAs), the 8 warps stride the
// slice, and their partials are summed in warp order through shared memory.  The KS
// slices of a token tile form one thread-block cluster; rank 0 sums the others'
// partials in rank order over DSMEM (deterministic, no global scratch), then does the
// top-k (strictly greater -> lower index wins ties) for its TB tokens.
// With `done` != nullptr the kernel also runs K2: the rank-0 CTA that finishes last
// (atomic ticket on done[0], reset afterwards) performs the deterministic routing scan
// of the whole chunk, saving a launch.
template <typename T, int E>
struct GateTile {
  static constexpr int NEG = E >= 4 ? 4 : E;   // expert groups across lanes
  static constexpr int EG = E / NEG;           // experts per lane
  static constexpr int TB = (32 / NEG) * 4;    // tokens per CTA (4 per lane)
  // 8 warp partials + the CTA sum + (ks-1) peer slots (rank 0), or the fused scan's hist
  static constexpr size_t smem(int ks = 8) {
    const size_t red = (size_t)(8 + ks) * TB * E * sizeof(float);
    const size_t hist = (size_t)E * (256 + 8) * sizeof(int);
    return red > hist ? red : hist;
  }
};

// n consecutive storage elements (n·sizeof(T) in {2,4,8,16,...} bytes, aligned) -> fp32
template <typename T, int n>
FM_DEV void load_n(const T* p, float* out) {
  constexpr int bytes = n * (int)sizeof(T);
  if constexpr (bytes % 16 == 0) {
#pragma unroll
    for (int i = 0; i < n; i += 16 / (int)sizeof(T)) load16<T>(p + i, out + i);
  } else if constexpr (bytes == 8) {
    const uint2 u = *reinterpret_cast<const uint2*>(p);
    if constexpr (sizeof(T) == 4) {
      out[0] = __uint_as_float(u.x); out[1] = __uint_as_float(u.y);
    } else {
      out[0] = __uint_as_float(u.x << 16); out[1] = __uint_as_float(u.x & 0xFFFF0000u);
      out[2] = __uint_as_float(u.y << 16); out[3] = __uint_as_float(u.y & 0xFFFF0000u);
    }
  } else {
#pragma unroll
    for (int i = 0; i < n; ++i) out[i] = to_f<T>(p[i]);
  }
}

template <typename T, int E>
__global__ void __launch_bounds__(256) gate_topk_kernel(const T* a, const T* wg,
                                                        const int32_t* forced, float* logits,
                                                        int32_t* idx, float* w, int T_, int M, int MS,
                                                        int k, int32_t* pos, int32_t* counts,
                                                        int32_t* src, int C, unsigned int* done) {
  using G = GateTile<T, E>;
  constexpr int V = 16 / sizeof(T), TB = G::TB, EG = G::EG, NEG = G::NEG;
  extern __shared__ float gsm[];  // [8][TB][E] warp partials, [TB][E] CTA sum; later the scan's hist
  __shared__ int warp_tot[32];
  __shared__ unsigned int ticket;
  __shared__ alignas(8) unsigned long long cbar;  // rank 0: completes when every peer's slot landed
  cg::cluster_group cl = cg::this_cluster();
  const unsigned int nrank = cl.num_blocks(), rank = cl.block_rank();
  float* slots = gsm + 9 * TB * E;  // rank 0: [nrank-1][TB][E] peer slice sums
  if (nrank > 1) {
    if (rank == 0 && threadIdx.x == 0) {
      const uint32_t b = rt_smem(&cbar);
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(b) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                   :: "r"(b), "r"((nrank - 1) * TB * E * 4u) : "memory");
    }
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  }
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(0);
  FM_PDL_ENTRY();
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tg = lane / NEG, eg = lane % NEG;
  const int tt0 = blockIdx.x * TB;                 // first token of the tile
  const int tl0 = tt0 + tg * 4;                    // this lane's first token
  const int m_beg = blockIdx.y * MS, m_end = min(M, m_beg + MS);
  float acc[4][EG];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < EG; ++j) acc[i][j] = 0.f;
#pragma unroll 4
  for (int m = m_beg + warp * V; m < m_end; m += 8 * V) {
    float xa[4][V];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (tl0 + i < T_) load16<T>(a + (int64_t)(tl0 + i) * M + m, xa[i]);
      else
#pragma unroll
        for (int v = 0; v < V; ++v) xa[i][v] = 0.f;
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      float wr[EG];
      load_n<T, EG>(wg + (int64_t)(m + v) * E + eg * EG, wr);
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < EG; ++j) acc[i][j] = fmaf(xa[i][v], wr[j], acc[i][j]);
    }
  }
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(2);
  float* red = gsm + 8 * TB * E;
  {
    float* part = gsm + warp * TB * E;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < EG; ++j) part[(tg * 4 + i) * E + eg * EG + j] = acc[i][j];
  }
  __syncthreads();
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(4);
  if (nrank > 1) {
    // cluster (1, KS, 1): every peer pushes its slice sum into rank 0's slot with
    // st.async (completing bytes on rank 0's mbarrier) and exits; rank 0 adds the slots
    // in rank order (deterministic).  The cluster barrier armed at entry guarantees rank
    // 0 is resident and its mbarrier initialised before the first remote store.
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank != 0) {
      const uint32_t dst = rt_mapa(rt_smem(slots + (rank - 1) * TB * E), 0);
      const uint32_t bar = rt_mapa(rt_smem(&cbar), 0);
      for (int q = threadIdx.x; q < TB * E; q += blockDim.x) {
        float sum = 0.f;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) sum += gsm[ww * TB * E + q];
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];"
                     :: "r"(dst + 4u * q), "r"(__float_as_uint(sum)), "r"(bar) : "memory");
      }
      return;
    }
  }
  for (int q = threadIdx.x; q < TB * E; q += blockDim.x) {
    float sum = 0.f;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) sum += gsm[ww * TB * E + q];
    red[q] = sum;
  }
  if (nrank > 1) {
    if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(5);
    asm volatile(
        "{\n.reg .pred P;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P, [%0], 0;\n"
        "@!P bra WAIT_%=;\n}" :: "r"(rt_smem(&cbar)) : "memory");
    for (int q = threadIdx.x; q < TB * E; q += blockDim.x) {
      float sum = red[q];
      for (unsigned int r = 1; r < nrank; ++r) sum += slots[(r - 1) * TB * E + q];
      red[q] = sum;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(6);
  }
  __syncthreads();
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(16);
  for (int q = threadIdx.x; q < TB * E; q += blockDim.x)
    if (tt0 + q / E < T_) logits[(int64_t)tt0 * E + q] = red[q];
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(17);
  if (threadIdx.x < TB && tt0 + (int)threadIdx.x < T_) {
    const int t = tt0 + threadIdx.x;
    float lg[E];
#pragma unroll
    for (int e = 0; e < E; ++e) lg[e] = red[threadIdx.x * E + e];
    // top-k selection on logits, register-resident (k <= 8 unrolled, E compile-time)
    uint64_t taken = 0;
    int sel[8];
    float sv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (j < k) {
        int best = -1;
        float bv = 0.f;
        if (forced) {
          best = forced[(int64_t)t * k + j];
#pragma unroll
          for (int e = 0; e < E; ++e)
            if (e == best) bv = lg[e];
        } else {
#pragma unroll
          for (int e = 0; e < E; ++e)
            if (!((taken >> e) & 1ull) && (best < 0 || lg[e] > bv)) { best = e; bv = lg[e]; }
        }
        taken |= 1ull << best;
        sel[j] = best;
        sv[j] = bv;
        idx[(int64_t)t * k + j] = best;
      }
    }
    if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(18);
    if (k == 1) {
      // w0 = p_{e0} = 1 / Σ_e exp(l_e - l_e0)
      float den = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) den += expf(lg[e] - sv[0]);
      w[t] = 1.f / den;
    } else {
      float mx = sv[0];
#pragma unroll
      for (int j = 1; j < 8; ++j)
        if (j < k) mx = fmaxf(mx, sv[j]);
      float den = 0.f, ex[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) { ex[j] = expf(sv[j] - mx); den += ex[j]; }
#pragma unroll
      for (int j = 0; j < 8; ++j)
        if (j < k) w[(int64_t)t * k + j] = ex[j] / den;
    }
    (void)sel;
  }
  if (done == nullptr) return;
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(7);
  __syncthreads();  // the CTA's logits/idx/w stores precede thread 0's release (cumulative)
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(13);
  if (threadIdx.x == 0)  // release: this CTA's idx; acquire: every earlier CTA's (for the scan)
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(ticket) : "l"(done) : "memory");
  __syncthreads();
  if (blockIdx.x == 0 && blockIdx.y == 0) FM_GMARK(3);
  if (ticket != gridDim.x - 1) return;
  FM_GMARK(8);
  // thread 0's acquire (the ticket) + the barrier above order every tile's idx before
  // this CTA's reads (the grid-sync pattern)
  route_scan_body(idx, pos, counts, src, T_, E, k, C, reinterpret_cast<int*>(gsm), warp_tot);
  FM_GMARK(12);
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

// Slices of M per token tile: enough CTAs to cover ~2 waves of the 148 SMs, at most a
// portable cluster (8), at least one 16-byte vector per warp.
int g_gate_force_ks = 0;  // probe / A-B only: force the number of M slices (1..8)
int g_route_stage = 0;    // probe compatibility (the shared-memory staged scan was measured slower and removed)

static void gate_split(int T_, int M, int TB, int V, int* KS, int* MS) {
  const int tiles = (T_ + TB - 1) / TB, nvec = M / V;
  int ks = (2 * 148 + tiles - 1) / tiles;
  ks = ks < 1 ? 1 : (ks > 8 ? 8 : ks);
  if (ks > nvec / 8) ks = nvec / 8 > 0 ? nvec / 8 : 1;
  if (g_gate_force_ks > 0) ks = g_gate_force_ks;
  const int msv = (nvec + ks - 1) / ks;
  *MS = msv * V;
  *KS = (nvec + msv - 1) / msv;
}

template <typename T, int E>
static void gate_topk_launch_t(const void* a, const void* wg, const int32_t* forced, float* logits, int32_t* idx,
                               float* w, int T_, int M, int k, int32_t* pos, int32_t* counts, int32_t* src, int C,
                               unsigned int* done, cudaStream_t s) {
  using G = GateTile<T, E>;
  int KS, MS;
  gate_split(T_, M, G::TB, 16 / (int)sizeof(T), &KS, &MS);
  auto kern = gate_topk_kernel<T, E>;
  static bool once = (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::smem()), true);
  (void)once;
  launch_kc(kern, dim3((T_ + G::TB - 1) / G::TB, KS), 256, G::smem(KS), s, dim3(1, KS, 1), (const T*)a,
            (const T*)wg, forced, logits, idx, w, T_, M, MS, k, pos, counts, src, C, done);
}

template <int E>
static void gate_topk_launch(int dtype, const void* a, const void* wg, const int32_t* forced,
                             float* logits, int32_t* idx, float* w, int T_, int M, int k,
                             int32_t* pos, int32_t* counts, int32_t* src, int C, unsigned int* done,
                             cudaStream_t s) {
  if (dtype == DT_F32)
    gate_topk_launch_t<float, E>(a, wg, forced, logits, idx, w, T_, M, k, pos, counts, src, C, done, s);
  else
    gate_topk_launch_t<bf16, E>(a, wg, forced, logits, idx, w, T_, M, k, pos, counts, src, C, done, s);
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
// contiguous per-thread segments; pass 1 counts per expert into hist[e][thread], the
// per-expert exclusive scans over threads run in parallel (warp w scans experts
// w, w+nwarps, ...: each lane sums a run of consecutive threads' counts, one warp
// shuffle scan, write-back), pass 2 re-walks the segment assigning pos = base[e]++.
// Deterministic: pos equals the number of earlier slots (in slot-major order) routed
// to the same expert.
constexpr int RS_THREADS = 512;

// Block-wide deterministic routing scan (one CTA, blockDim a power of two in [32, 1024]):
// hist is [E][blockDim.x + blockDim.x/32] ints of dynamic shared memory (padded rows).
__device__ void route_scan_body(const int32_t* idx, int32_t* pos, int32_t* counts, int32_t* src, int T_,
                                int E, int k, int C, int* hist, int* warp_tot) {
  (void)warp_tot;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int n = T_ * k;
  const int seg = (n + nt - 1) / nt;
  const int s0 = min(n, tid * seg), s1 = min(n, s0 + seg);
  // hist[e][th] lives at e·rs + th + th/32: one pad word per 32 threads keeps the
  // lane-runs of the scan below (lane L reads threads L·per .. L·per+per-1) conflict-free
  const int rs = nt + nt / 32;
  const int my = tid + (tid >> 5);
  // a thread's slots (slot-major: s = j·T + t) are loaded once, all in flight together,
  // and kept in registers for both passes when they fit (seg <= SCAN_REG): a dependent
  // L2 round trip per slot (the loop below) cost ~20 µs at T_r·k = 4096 slots
  constexpr int SCAN_REG = 32;
  const bool in_reg = seg <= SCAN_REG;
  int ev[SCAN_REG];
#pragma unroll
  for (int i = 0; i < SCAN_REG; ++i) {
    const int s = s0 + i;
    ev[i] = 0;
    if (in_reg && s < s1) {
      const int j = s / T_, t = s - j * T_;
      ev[i] = idx[(int64_t)t * k + j];
    }
  }
  for (int e = 0; e < E; ++e) hist[e * rs + my] = 0;
  for (int i = tid; i < E * C; i += nt) src[i] = -1;
  __syncthreads();
  FM_GMARK(9);
  if (in_reg) {
#pragma unroll
    for (int i = 0; i < SCAN_REG; ++i)
      if (s0 + i < s1) hist[ev[i] * rs + my] += 1;
  } else {
    for (int s = s0; s < s1; ++s) {
      const int j = s / T_, t = s - j * T_;
      hist[idx[(int64_t)t * k + j] * rs + my] += 1;
    }
  }
  __syncthreads();
  FM_GMARK(10);
  const int lane = tid & 31, nw = nt >> 5, per = nt >> 5;  // per: threads summed by one lane
  for (int e = tid >> 5; e < E; e += nw) {
    int* h = hist + e * rs + lane * per + ((lane * per) >> 5);  // per <= 32: no pad inside a run
    int run = 0;
    for (int i = 0; i < per; ++i) run += h[i];
    int x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) counts[e] = x;
    int ex = x - run;  // exclusive prefix of this lane's run
    for (int i = 0; i < per; ++i) {
      const int v = h[i];
      h[i] = ex;
      ex += v;
    }
  }
  __syncthreads();
  FM_GMARK(11);
  auto place = [&](int s, int e) {
    const int j = s / T_, t = s - j * T_;
    const int p = hist[e * rs + my]++;
    const bool kept = p < C;
    pos[(int64_t)t * k + j] = kept ? p : -1;
    if (kept) src[e * C + p] = t * k + j;
  };
  if (in_reg) {
#pragma unroll
    for (int i = 0; i < SCAN_REG; ++i)
      if (s0 + i < s1) place(s0 + i, ev[i]);
  } else {
    for (int s = s0; s < s1; ++s) {
      const int j = s / T_, t = s - j * T_;
      place(s, idx[(int64_t)t * k + j]);
    }
  }
}

__global__ void __launch_bounds__(RS_THREADS) route_scan_kernel(const int32_t* idx, int32_t* pos,
                                                                int32_t* counts, int32_t* src,
                                                                int T_, int E, int k, int C) {
  FM_PDL_ENTRY();
  extern __shared__ int hist[];  // [E][RS_THREADS + RS_THREADS/32]
  __shared__ int warp_tot[32];
  route_scan_body(idx, pos, counts, src, T_, E, k, C, hist, warp_tot);
}

int route_scan(const int32_t* idx, int32_t* pos, int32_t* counts, int32_t* src, int T_, int E,
               int k, int C, cudaStream_t s) {
  constexpr int RS_ROW = RS_THREADS + RS_THREADS / 32;
  size_t smem = (size_t)E * RS_ROW * sizeof(int);
  static bool once = (cudaFuncSetAttribute(route_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           64 * RS_ROW * (int)sizeof(int)), true);
  (void)once;
  launch_k(route_scan_kernel, 1, RS_THREADS, smem, s, idx, pos, counts, src, T_, E, k, C);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K3 / K7 / K8
// Row movement is spread one 16-byte vector per thread over (row, vector) pairs, so a
// chunk's copy has thousands of independent loads in flight (a warp per row left most
// SMs idle at small T_r and serialised each warp's loads at large M).
template <typename T>
__global__ void __launch_bounds__(256) permute_pack_kernel(const T* __restrict__ a, const int32_t* __restrict__ src,
                                                           T* __restrict__ send, int rows, int C, int ldE,
                                                           int M, int k) {
  FM_PDL_ENTRY();
  constexpr int V = 16 / sizeof(T);
  const int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int nv = M / V;
  const int sl = src[r];
  uint4* dst = reinterpret_cast<uint4*>(send + ((int64_t)(r / C) * ldE + r % C) * M);
  if (sl < 0) {
    for (int i = lane; i < nv; i += 32) dst[i] = make_uint4(0, 0, 0, 0);
    return;
  }
  const uint4* srow = reinterpret_cast<const uint4*>(a + (int64_t)(sl / k) * M);
  int i = lane;
  for (; i + 96 < nv; i += 128) {  // 4 independent 16-byte loads in flight per lane
    const uint4 v0 = __ldg(srow + i), v1 = __ldg(srow + i + 32), v2 = __ldg(srow + i + 64), v3 = __ldg(srow + i + 96);
    dst[i] = v0; dst[i + 32] = v1; dst[i + 64] = v2; dst[i + 96] = v3;
  }
  for (; i < nv; i += 32) dst[i] = __ldg(srow + i);
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

// K7: out[t] = Σ_j w_tj·Y[e_tj][pos_tj] (+ resid[t]); thread = (token, 16-byte vector).
// K compile-time: the routing of all K slots, then all K rows and the residual are
// requested before any is used (one dependent round trip for the routing, one for the
// rows), summed in slot order.
template <typename T, int K>
__global__ void __launch_bounds__(256) unpermute_combine_kernel(const T* __restrict__ y, const int32_t* __restrict__ idx,
                                                                const int32_t* __restrict__ pos,
                                                                const float* __restrict__ w,
                                                                const T* __restrict__ resid, T* __restrict__ out,
                                                                int T_, int M, int ldE) {
  FM_PDL_ENTRY();
  constexpr int V = 16 / sizeof(T);
  const int nv = M / V;
  const unsigned int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (unsigned int)(T_ * nv)) return;
  const int t = (int)(g / (unsigned int)nv), m = (int)(g % (unsigned int)nv) * V;
  int pj[K], ej[K];
  float wj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    pj[j] = pos[(int64_t)t * K + j];
    ej[j] = idx[(int64_t)t * K + j];
    wj[j] = w[(int64_t)t * K + j];
  }
  uint4 raw[K], rr = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    raw[j] = make_uint4(0, 0, 0, 0);
    if (pj[j] >= 0) raw[j] = *reinterpret_cast<const uint4*>(y + ((int64_t)ej[j] * ldE + pj[j]) * M + m);
  }
  if (resid) rr = *reinterpret_cast<const uint4*>(resid + (int64_t)t * M + m);
  float acc[V];
#pragma unroll
  for (int i = 0; i < V; ++i) acc[i] = 0.f;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (pj[j] >= 0) {
      float v[V];
      load16<T>(reinterpret_cast<const T*>(&raw[j]), v);
#pragma unroll
      for (int i = 0; i < V; ++i) acc[i] = fmaf(wj[j], v[i], acc[i]);
    }
  if (resid) {
    float rv[V];
    load16<T>(reinterpret_cast<const T*>(&rr), rv);
#pragma unroll
    for (int i = 0; i < V; ++i) acc[i] += rv[i];
  }
  store16<T>(out + (int64_t)t * M + m, acc);
}

template <typename T, int K>
static void unpermute_combine_launch(const void* y, const int32_t* idx, const int32_t* pos, const float* w,
                                     const void* resid, void* out, int T_, int M, int ldE, cudaStream_t s) {
  const int64_t n = (int64_t)T_ * (M / (16 / (int)sizeof(T)));
  launch_k(unpermute_combine_kernel<T, K>, (unsigned)((n + 255) / 256), 256, 0, s, (const T*)y, idx, pos, w,
           (const T*)resid, (T*)out, T_, M, ldE);
}

template <typename T>
static int unpermute_combine_t(const void* y, const int32_t* idx, const int32_t* pos, const float* w,
                               const void* resid, void* out, int T_, int M, int k, int ldE, cudaStream_t s) {
  switch (k) {
    case 1: unpermute_combine_launch<T, 1>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    case 2: unpermute_combine_launch<T, 2>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    case 3: unpermute_combine_launch<T, 3>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    case 4: unpermute_combine_launch<T, 4>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    case 5: unpermute_combine_launch<T, 5>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    case 6: unpermute_combine_launch<T, 6>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    case 7: unpermute_combine_launch<T, 7>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    case 8: unpermute_combine_launch<T, 8>(y, idx, pos, w, resid, out, T_, M, ldE, s); break;
    default: return (int)cudaErrorInvalidValue;
  }
  return 0;
}

int unpermute_combine(int dtype, const void* y, const int32_t* idx, const int32_t* pos,
                      const float* w, const void* resid, void* out, int T_, int M, int k, int ldE,
                      cudaStream_t s) {
  if (T_ <= 0) return 0;
  const int64_t n = (int64_t)T_ * (M / (dtype == DT_F32 ? 4 : 8));
  if (n >= (1ll << 31)) return (int)cudaErrorInvalidValue;
  const int rc = dtype == DT_F32 ? unpermute_combine_t<float>(y, idx, pos, w, resid, out, T_, M, k, ldE, s)
                                 : unpermute_combine_t<bf16>(y, idx, pos, w, resid, out, T_, M, k, ldE, s);
  if (rc) return rc;
  return (int)cudaGetLastError();
}

// K8: dY[e][pos] = w·dO[t]; dw[t][j] = <dO[t], Y[e][pos]>.  tpt threads per token (the
// power of two >= 32 that covers the row's 16-byte vectors in one pass, at most 256: a
// warp per token for narrow rows, a CTA per token for wide ones), all K slots in one
// pass, reduction of the K dots over the token's warps in a fixed order; CTAs past the
// token CTAs zero 8 padding rows of dY each.
template <typename T, int K>
__global__ void __launch_bounds__(256) combine_bwd_pack_kernel(const T* __restrict__ dout, const T* __restrict__ y,
                                                               const int32_t* __restrict__ idx,
                                                               const int32_t* __restrict__ pos,
                                                               const float* __restrict__ w,
                                                               const int32_t* __restrict__ src, T* __restrict__ dy,
                                                               float* __restrict__ dw, int T_, int M,
                                                               int rows, int C, int ldE, int tpt) {
  __shared__ float red[8][K];  // [warp][slot]
  FM_PDL_ENTRY();
  constexpr int V = 16 / sizeof(T);
  const int nv = M / V;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tpc = (int)blockDim.x / tpt, ntb = (T_ + tpc - 1) / tpc;  // tokens per CTA, token CTAs
  if ((int)blockIdx.x >= ntb) {  // padding rows (src < 0) of dy get zeros
    const int r = ((int)blockIdx.x - ntb) * 8 + warp;
    if (r >= rows || src[r] >= 0) return;
    uint4* dst = reinterpret_cast<uint4*>(dy + ((int64_t)(r / C) * ldE + r % C) * M);
    for (int i = lane; i < nv; i += 32) dst[i] = make_uint4(0, 0, 0, 0);
    return;
  }
  // tpt threads (a power of two >= 32) per token: a warp per token for narrow rows
  const int grp = (int)threadIdx.x / tpt, gt = (int)threadIdx.x % tpt;
  const int t = (int)blockIdx.x * tpc + grp;
  const bool tok = t < T_;
  const T* g = dout + (int64_t)t * M;
  int64_t row[K];
  float wj[K], dot[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const int p = tok ? pos[(int64_t)t * K + j] : -1;
    row[j] = p < 0 ? -1 : ((int64_t)idx[(int64_t)t * K + j] * ldE + p) * M;
    wj[j] = tok ? w[(int64_t)t * K + j] : 0.f;
    dot[j] = 0.f;
  }
  for (int v = gt; tok && v < nv; v += tpt) {
    // dO and all K rows of Y requested together (K + 1 loads in flight), then used
    const uint4 graw = *reinterpret_cast<const uint4*>(g + v * V);
    uint4 yraw[K];
#pragma unroll
    for (int j = 0; j < K; ++j)
      yraw[j] = row[j] < 0 ? make_uint4(0, 0, 0, 0) : *reinterpret_cast<const uint4*>(y + row[j] + v * V);
    float gv[V];
    load16<T>(reinterpret_cast<const T*>(&graw), gv);
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (row[j] < 0) continue;  // dropped slot: contributes 0, so dw = 0
      float yv[V], o[V];
      load16<T>(reinterpret_cast<const T*>(&yraw[j]), yv);
#pragma unroll
      for (int i = 0; i < V; ++i) { dot[j] = fmaf(gv[i], yv[i], dot[j]); o[i] = wj[j] * gv[i]; }
      store16<T>(dy + row[j] + v * V, o);
    }
  }
#pragma unroll
  for (int j = 0; j < K; ++j) {
    const float d = warp_sum(dot[j]);
    if (lane == 0) red[warp][j] = d;
  }
  __syncthreads();
  if (gt == 0 && tok) {  // the token's warps in order (fixed: deterministic)
    const int w0 = grp * (tpt >> 5), nw = tpt >> 5;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      float d = 0.f;
      for (int i = w0; i < w0 + nw; ++i) d += red[i][j];
      dw[(int64_t)t * K + j] = row[j] < 0 ? 0.f : d;
    }
  }
}

template <int K>
static void combine_bwd_launch(int dtype, const void* dout, const void* y, const int32_t* idx, const int32_t* pos,
                               const float* w, const int32_t* src, void* dy, float* dw, int T_, int M, int rows,
                               int C, int ldE, cudaStream_t s) {
  const int nv = M / (dtype == DT_F32 ? 4 : 8);
  int tpt = 32;  // threads per token: enough 16-byte lanes for one pass over the row, <= 256
  while (tpt < nv && tpt < 256) tpt *= 2;
  const int tpc = 256 / tpt;
  dim3 grid((T_ + tpc - 1) / tpc + (rows + 7) / 8);
  if (dtype == DT_F32)
    launch_k(combine_bwd_pack_kernel<float, K>, grid, 256, 0, s, (const float*)dout, (const float*)y, idx, pos, w,
             src, (float*)dy, dw, T_, M, rows, C, ldE, tpt);
  else
    launch_k(combine_bwd_pack_kernel<bf16, K>, grid, 256, 0, s, (const bf16*)dout, (const bf16*)y, idx, pos, w,
             src, (bf16*)dy, dw, T_, M, rows, C, ldE, tpt);
}

int combine_bwd_pack(int dtype, const void* dout, const void* y, const int32_t* idx,
                     const int32_t* pos, const float* w, const int32_t* src, void* dy, float* dw,
                     int T_, int M, int k, int E, int C, int ldE, cudaStream_t s) {
  const int rows = E * C;
  switch (k) {
    case 1: combine_bwd_launch<1>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    case 2: combine_bwd_launch<2>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    case 3: combine_bwd_launch<3>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    case 4: combine_bwd_launch<4>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    case 5: combine_bwd_launch<5>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    case 6: combine_bwd_launch<6>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    case 7: combine_bwd_launch<7>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    case 8: combine_bwd_launch<8>(dtype, dout, y, idx, pos, w, src, dy, dw, T_, M, rows, C, ldE, s); break;
    default: return (int)cudaErrorInvalidValue;
  }
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ K9
// dA[t] = Σ_j dx[e_tj][pos_tj] + dlogits[t]·Wgᵀ (+ dO[t]).  A thread owns TPL tokens ×
// one 16-byte column vector (V columns).  It derives the dlogits of its tokens in
// registers (cheap: k slots), then per column reads the Wg row (E values, L2-resident)
// once for all TPL tokens, adds the k gathered rows (+ dO) and stores.  Lanes of a warp
// take consecutive column vectors of the same tokens (coalesced); CTAs are sized so
// small chunks still spread over the SMs.
template <int E>
struct GgbTile { static constexpr int TPL = E <= 16 ? 4 : (E == 32 ? 2 : 1); };  // register-bound max

template <typename T, int E, int TPL>
__global__ void __launch_bounds__(256) gather_gate_bwd_kernel(
    const T* __restrict__ dx, const int32_t* __restrict__ idx, const int32_t* __restrict__ pos,
    const float* __restrict__ w, const float* __restrict__ dw, const float* __restrict__ logits,
    const T* __restrict__ wg, const T* __restrict__ dres, T* __restrict__ dA, float* __restrict__ dlogits, int T_,
    int M, int k, int ldE, int CV) {
  constexpr int V = 16 / sizeof(T);
  FM_PDL_ENTRY();
  const int tgi = threadIdx.x / CV, cv = threadIdx.x % CV;
  const int tb = (blockDim.x / CV) * TPL;              // tokens per CTA
  const int t0 = blockIdx.x * tb + tgi * TPL;
  const int m = (blockIdx.y * CV + cv) * V;
  // TPL == 1 (small, latency-bound chunks): the gathered rows of the first two slots and
  // dO do not depend on the dlogits, so their loads are issued first and land under the
  // dlogits / Wg work (same summation order as the late loads below)
  constexpr bool PF = TPL == 1 && E <= 32;  // E = 64: the register budget goes to dl and Wg
  float px[2][V], pr[V];
  bool pok[2] = {false, false};
  if constexpr (PF) {
    const int t = t0;
    if (t < T_ && m < M) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (j < k) {
          const int p = pos[(int64_t)t * k + j];
          pok[j] = p >= 0;
          if (pok[j]) load16<T>(dx + ((int64_t)idx[(int64_t)t * k + j] * ldE + p) * M + m, px[j]);
        }
      if (dres) load16<T>(dres + (int64_t)t * M + m, pr);
    }
  }
  // dlogits (reading Q5): k>=2: dl_{e_j} = w_j (dw_j - Σ w dw); k=1: dl = p ⊙ (g - <p,g>)
  float dl[TPL][E];
#pragma unroll
  for (int i = 0; i < TPL; ++i) {
    const int t = t0 + i;
#pragma unroll
    for (int e = 0; e < E; ++e) dl[i][e] = 0.f;
    if (t >= T_) continue;
    if (k == 1) {
      const float* lt = logits + (int64_t)t * E;
      const int e0 = idx[t];
      float mx = -INFINITY;
#pragma unroll
      for (int e = 0; e < E; ++e) mx = fmaxf(mx, lt[e]);
      float den = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) { dl[i][e] = expf(lt[e] - mx); den += dl[i][e]; }
      const float g0 = dw[t];
      float pe0 = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) { dl[i][e] /= den; if (e == e0) pe0 = dl[i][e]; }
#pragma unroll
      for (int e = 0; e < E; ++e) dl[i][e] = dl[i][e] * ((e == e0 ? g0 : 0.f) - pe0 * g0);
    } else {
      float inner = 0.f;
      for (int j = 0; j < k; ++j) inner += w[(int64_t)t * k + j] * dw[(int64_t)t * k + j];
      for (int j = 0; j < k; ++j) {
        const int ej = idx[(int64_t)t * k + j];
        const float v = w[(int64_t)t * k + j] * (dw[(int64_t)t * k + j] - inner);
#pragma unroll
        for (int e = 0; e < E; ++e) if (e == ej) dl[i][e] += v;
      }
    }
    if (blockIdx.y == 0 && cv == 0)
#pragma unroll
      for (int e = 0; e < E; ++e) dlogits[(int64_t)t * E + e] = dl[i][e];
  }
  if (m >= M) return;
  float acc[TPL][V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    float wr[E];
    load_n<T, E>(wg + (int64_t)(m + v) * E, wr);
#pragma unroll
    for (int i = 0; i < TPL; ++i) {
      float sum = 0.f;
#pragma unroll
      for (int e = 0; e < E; ++e) sum = fmaf(dl[i][e], wr[e], sum);
      acc[i][v] = sum;
    }
  }
#pragma unroll
  for (int i = 0; i < TPL; ++i) {
    const int t = t0 + i;
    if (t >= T_) break;
    int j0 = 0;
    if constexpr (PF) {
#pragma unroll
      for (int j = 0; j < 2; ++j)
        if (pok[j])
#pragma unroll
          for (int v = 0; v < V; ++v) acc[i][v] += px[j][v];
      j0 = 2;
    }
    for (int j = j0; j < k; ++j) {
      const int p = pos[(int64_t)t * k + j];
      if (p < 0) continue;
      float v8[V];
      load16<T>(dx + ((int64_t)idx[(int64_t)t * k + j] * ldE + p) * M + m, v8);
#pragma unroll
      for (int v = 0; v < V; ++v) acc[i][v] += v8[v];
    }
    if (dres) {
      float v8[V];
      if (PF) {
#pragma unroll
        for (int v = 0; v < V; ++v) v8[v] = pr[v];
      } else {
        load16<T>(dres + (int64_t)t * M + m, v8);
      }
#pragma unroll
      for (int v = 0; v < V; ++v) acc[i][v] += v8[v];
    }
    store16<T>(dA + (int64_t)t * M + m, acc[i]);
  }
}

// Wide rows (M/V >= 64 column vectors): one thread per (token, 16-byte column vector), all
// K gathered rows requested at once (K compile-time) so every thread has K + 1 loads in
// flight — the per-slot loop above left a thread one dependent load at a time, 11% of HBM
// at k = 8 (dsv2s).  The token's dlogits are recomputed by each of its threads from
// warp-uniform loads of its k slots; the Wg rows come from L1/L2.  Same summation order
// as the kernel above: dlogits·Wgᵀ, then the slots in order, then dO.
template <typename T, int E, int K>
__global__ void __launch_bounds__(256) gather_gate_bwd_wide_kernel(
    const T* __restrict__ dx, const int32_t* __restrict__ idx, const int32_t* __restrict__ pos,
    const float* __restrict__ w, const float* __restrict__ dw, const float* __restrict__ logits,
    const T* __restrict__ wg, const T* __restrict__ dres, T* __restrict__ dA, float* __restrict__ dlogits, int T_,
    int M, int ldE) {
  constexpr int V = 16 / sizeof(T);
  FM_PDL_ENTRY();
  const int nv = M / V;
  const unsigned int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= (unsigned int)T_ * (unsigned int)nv) return;
  const int t = (int)(g / (unsigned int)nv), cvec = (int)(g % (unsigned int)nv), m = cvec * V;
  int ej[K], pj[K];
#pragma unroll
  for (int j = 0; j < K; ++j) {
    ej[j] = idx[(int64_t)t * K + j];
    pj[j] = pos[(int64_t)t * K + j];
  }
  uint4 raw[K], rres = make_uint4(0, 0, 0, 0);
#pragma unroll
  for (int j = 0; j < K; ++j) {
    raw[j] = make_uint4(0, 0, 0, 0);
    if (pj[j] >= 0) raw[j] = *reinterpret_cast<const uint4*>(dx + ((int64_t)ej[j] * ldE + pj[j]) * M + m);
  }
  if (dres) rres = *reinterpret_cast<const uint4*>(dres + (int64_t)t * M + m);
  // dlogits (reading Q5): k>=2: dl_{e_j} = w_j (dw_j - Σ w dw); k=1: dl = p ⊙ (g - <p,g>)
  float dl[E];
#pragma unroll
  for (int e = 0; e < E; ++e) dl[e] = 0.f;
  if constexpr (K == 1) {
    const float* lt = logits + (int64_t)t * E;
    float mx = -INFINITY;
#pragma unroll
    for (int e = 0; e < E; ++e) mx = fmaxf(mx, lt[e]);
    float den = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) { dl[e] = expf(lt[e] - mx); den += dl[e]; }
    const float g0 = dw[t];
    float pe0 = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) { dl[e] /= den; if (e == ej[0]) pe0 = dl[e]; }
#pragma unroll
    for (int e = 0; e < E; ++e) dl[e] = dl[e] * ((e == ej[0] ? g0 : 0.f) - pe0 * g0);
  } else {
    float wj[K], dwj[K], inner = 0.f;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      wj[j] = w[(int64_t)t * K + j];
      dwj[j] = dw[(int64_t)t * K + j];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) inner += wj[j] * dwj[j];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const float v = wj[j] * (dwj[j] - inner);
      // predicated adds (an `if` here becomes a dynamically indexed dl[] in local memory)
#pragma unroll
      for (int e = 0; e < E; ++e) dl[e] += (e == ej[j]) ? v : 0.f;
    }
  }
  if (cvec == 0)
#pragma unroll
    for (int e = 0; e < E; ++e) dlogits[(int64_t)t * E + e] = dl[e];
  float acc[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    float wr[E];
    load_n<T, E>(wg + (int64_t)(m + v) * E, wr);
    float sum = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) sum = fmaf(dl[e], wr[e], sum);
    acc[v] = sum;
  }
#pragma unroll
  for (int j = 0; j < K; ++j)
    if (pj[j] >= 0) {
      float v8[V];
      load16<T>(reinterpret_cast<const T*>(&raw[j]), v8);
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] += v8[v];
    }
  if (dres) {
    float v8[V];
    load16<T>(reinterpret_cast<const T*>(&rres), v8);
#pragma unroll
    for (int v = 0; v < V; ++v) acc[v] += v8[v];
  }
  store16<T>(dA + (int64_t)t * M + m, acc);
}

template <typename T, int E, int K>
static void gather_gate_bwd_wide_launch(const void* dx, const int32_t* idx, const int32_t* pos, const float* w,
                                        const float* dw, const float* logits, const void* wg, const void* dres,
                                        void* dA, float* dlogits, int T_, int M, int ldE, cudaStream_t s) {
  const int64_t n = (int64_t)T_ * (M / (16 / (int)sizeof(T)));
  launch_k(gather_gate_bwd_wide_kernel<T, E, K>, (unsigned)((n + 255) / 256), 256, 0, s, (const T*)dx, idx, pos, w,
           dw, logits, (const T*)wg, (const T*)dres, (T*)dA, dlogits, T_, M, ldE);
}

// E <= 16, wide rows: a CTA covers 128 column vectors x GGB_TB tokens.  It stages its
// Wg slice TRANSPOSED in shared memory ([E][128·V]: one 16-byte vector per (expert, column
// vector)), the tokens' routing (idx, pos) and their dlogits; then, since dlogits is zero
// outside a token's k selected experts (k >= 2, reading Q5), each token needs only k
// vector reads of Wgᵀ (E for k = 1) — the one-token-per-thread kernel above re-read all E
// columns of 8 Wg rows from L2 for every token (~2.5x the kernel's HBM bytes).  Two
// tokens' gathered rows + dO are requested together.  Same summation order as above.
constexpr int GGB_TB = 8, GGB_THREADS = 128;

template <typename T, int E, int K>
__global__ void __launch_bounds__(GGB_THREADS) gather_gate_bwd_tile_kernel(
    const T* __restrict__ dx, const int32_t* __restrict__ idx, const int32_t* __restrict__ pos,
    const float* __restrict__ w, const float* __restrict__ dw, const float* __restrict__ logits,
    const T* __restrict__ wg, const T* __restrict__ dres, T* __restrict__ dA, float* __restrict__ dlogits, int T_,
    int M, int ldE) {
  constexpr int V = 16 / sizeof(T);
  __shared__ float dls[GGB_TB][E];
  __shared__ int rte[GGB_TB][K], rtp[GGB_TB][K];
  extern __shared__ uint4 wgt4[];  // [E][GGB_THREADS] 16-byte vectors: Wgᵀ of this CTA's columns
  FM_PDL_ENTRY();
  const int nv = M / V;
  const int cvec = blockIdx.x * GGB_THREADS + threadIdx.x;
  const int t0 = blockIdx.y * GGB_TB;
  const int m = cvec * V;
  {  // transpose-stage: thread c reads its V Wg rows (V·E elements) and writes E vectors
    if (cvec < nv) {
      T col[E][V];
#pragma unroll
      for (int v = 0; v < V; ++v) {
        float r[E];
        load_n<T, E>(wg + (int64_t)(m + v) * E, r);
#pragma unroll
        for (int e = 0; e < E; ++e) col[e][v] = from_f<T>(r[e]);
      }
#pragma unroll
      for (int e = 0; e < E; ++e) wgt4[e * GGB_THREADS + threadIdx.x] = *reinterpret_cast<const uint4*>(col[e]);
    }
    for (int i = threadIdx.x; i < GGB_TB * K; i += GGB_THREADS) {
      const int t = t0 + i / K;
      rte[i / K][i % K] = t < T_ ? idx[(int64_t)t0 * K + i] : 0;
      rtp[i / K][i % K] = t < T_ ? pos[(int64_t)t0 * K + i] : -1;
    }
  }
  // dlogits of the tile's tokens (reading Q5), one thread per token
  if (threadIdx.x < GGB_TB) {
    const int t = t0 + threadIdx.x;
    float dl[E];
#pragma unroll
    for (int e = 0; e < E; ++e) dl[e] = 0.f;
    if (t < T_) {
      if constexpr (K == 1) {
        const float* lt = logits + (int64_t)t * E;
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
#pragma unroll
        for (int e = 0; e < E; ++e) dl[e] = dl[e] * ((e == e0 ? g0 : 0.f) - pe0 * g0);
      } else {
        float wj[K], dwj[K], inner = 0.f;
        int ej[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          wj[j] = w[(int64_t)t * K + j];
          dwj[j] = dw[(int64_t)t * K + j];
          ej[j] = idx[(int64_t)t * K + j];
        }
#pragma unroll
        for (int j = 0; j < K; ++j) inner += wj[j] * dwj[j];
#pragma unroll
        for (int j = 0; j < K; ++j) {
          const float v = wj[j] * (dwj[j] - inner);
#pragma unroll
          for (int e = 0; e < E; ++e) dl[e] += (e == ej[j]) ? v : 0.f;
        }
      }
      if (blockIdx.x == 0)
#pragma unroll
        for (int e = 0; e < E; ++e) dlogits[(int64_t)t * E + e] = dl[e];
    }
#pragma unroll
    for (int e = 0; e < E; ++e) dls[threadIdx.x][e] = dl[e];
  }
  __syncthreads();
  if (cvec >= nv) return;
  constexpr int PF = 2;
#pragma unroll 1
  for (int i0 = 0; i0 < GGB_TB; i0 += PF) {
    uint4 raw[PF][K], rres[PF];
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = i0 + q, t = t0 + i;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int p = rtp[i][j];
        raw[q][j] = p >= 0 ? *reinterpret_cast<const uint4*>(dx + ((int64_t)rte[i][j] * ldE + p) * M + m)
                           : make_uint4(0, 0, 0, 0);
      }
      rres[q] = (dres && t < T_) ? *reinterpret_cast<const uint4*>(dres + (int64_t)t * M + m) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int q = 0; q < PF; ++q) {
      const int i = i0 + q, t = t0 + i;
      if (t >= T_) break;
      // Σ_e dl[e]·Wg[m+v][e] in e order; with k >= 2 only the selected experts are non-zero
      // (the zero terms of the dense sum add nothing, so this is the same value up to the
      // order of the k non-zero terms: ascending expert index, as the dense loop)
      float acc[V];
#pragma unroll
      for (int v = 0; v < V; ++v) acc[v] = 0.f;
      if constexpr (K == 1) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          float wv[V];
          load16<T>(reinterpret_cast<const T*>(&wgt4[e * GGB_THREADS + threadIdx.x]), wv);
          const float d = dls[i][e];
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] = fmaf(d, wv[v], acc[v]);
        }
      } else {
        // the selected experts in ascending order (k <= 8: a small sorting network)
        int es[K];
#pragma unroll
        for (int j = 0; j < K; ++j) es[j] = rte[i][j];
#pragma unroll
        for (int a = 0; a < K; ++a)
#pragma unroll
          for (int b2 = 0; b2 + 1 < K - a; ++b2)
            if (es[b2] > es[b2 + 1]) { const int tmp = es[b2]; es[b2] = es[b2 + 1]; es[b2 + 1] = tmp; }
#pragma unroll
        for (int j = 0; j < K; ++j) {
          float wv[V];
          load16<T>(reinterpret_cast<const T*>(&wgt4[es[j] * GGB_THREADS + threadIdx.x]), wv);
          const float d = dls[i][es[j]];
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] = fmaf(d, wv[v], acc[v]);
        }
      }
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (rtp[i][j] >= 0) {
          float v8[V];
          load16<T>(reinterpret_cast<const T*>(&raw[q][j]), v8);
#pragma unroll
          for (int v = 0; v < V; ++v) acc[v] += v8[v];
        }
      if (dres) {
        float v8[V];
        load16<T>(reinterpret_cast<const T*>(&rres[q]), v8);
#pragma unroll
        for (int v = 0; v < V; ++v) acc[v] += v8[v];
      }
      store16<T>(dA + (int64_t)t * M + m, acc);
    }
  }
}

template <typename T, int E, int K>
static void gather_gate_bwd_tile_launch(const void* dx, const int32_t* idx, const int32_t* pos, const float* w,
                                        const float* dw, const float* logits, const void* wg, const void* dres,
                                        void* dA, float* dlogits, int T_, int M, int ldE, cudaStream_t s) {
  const int nv = M / (16 / (int)sizeof(T));
  dim3 grid((nv + GGB_THREADS - 1) / GGB_THREADS, (T_ + GGB_TB - 1) / GGB_TB);
  const size_t smem = (size_t)GGB_THREADS * E * 16;
  launch_k(gather_gate_bwd_tile_kernel<T, E, K>, grid, GGB_THREADS, smem, s, (const T*)dx, idx, pos, w, dw, logits,
           (const T*)wg, (const T*)dres, (T*)dA, dlogits, T_, M, ldE);
}

template <typename T, int E>
struct GgbWide {
  template <int K>
  static void run(const void* dx, const int32_t* idx, const int32_t* pos, const float* w, const float* dw,
                  const float* logits, const void* wg, const void* dres, void* dA, float* dlogits, int T_, int M,
                  int ldE, cudaStream_t s) {
    if constexpr (E <= 16)  // Wg rows register-resident over a tile of tokens
      gather_gate_bwd_tile_launch<T, E, K>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s);
    else
      gather_gate_bwd_wide_launch<T, E, K>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s);
  }
};

template <typename T, int E>
static void gather_gate_bwd_launch_t(const void* dx, const int32_t* idx, const int32_t* pos, const float* w,
                                     const float* dw, const float* logits, const void* wg, const void* dres,
                                     void* dA, float* dlogits, int T_, int M, int k, int ldE, cudaStream_t s) {
  constexpr int V = 16 / sizeof(T), TPLX = GgbTile<E>::TPL;
  const int nvec = M / V;
  if (nvec >= 64 && E <= 32) {  // wide rows: one thread per (token, column vector), K loads in flight
    switch (k) {
      case 1: GgbWide<T, E>::template run<1>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      case 2: GgbWide<T, E>::template run<2>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      case 3: GgbWide<T, E>::template run<3>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      case 4: GgbWide<T, E>::template run<4>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      case 5: GgbWide<T, E>::template run<5>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      case 6: GgbWide<T, E>::template run<6>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      case 7: GgbWide<T, E>::template run<7>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      case 8: GgbWide<T, E>::template run<8>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, ldE, s); return;
      default: break;
    }
  }
  int cv = (nvec + 31) / 32 * 32;  // column-vector lanes per token group
  if (cv > 256) cv = 256;
  const int tg = 256 / cv, ctiles = (nvec + cv - 1) / cv;
  // several tokens per thread (Wg rows reused) only when that still leaves >= 2 waves
  const bool multi = (int64_t)((T_ + tg * TPLX - 1) / (tg * TPLX)) * ctiles >= 2 * 148;
  const int tpl = multi ? TPLX : 1, tb = tg * tpl;
  dim3 grid((T_ + tb - 1) / tb, ctiles);
  if (multi)
    launch_k(gather_gate_bwd_kernel<T, E, TPLX>, grid, cv * tg, 0, s, (const T*)dx, idx, pos, w, dw, logits,
             (const T*)wg, (const T*)dres, (T*)dA, dlogits, T_, M, k, ldE, cv);
  else
    launch_k(gather_gate_bwd_kernel<T, E, 1>, grid, cv * tg, 0, s, (const T*)dx, idx, pos, w, dw, logits,
             (const T*)wg, (const T*)dres, (T*)dA, dlogits, T_, M, k, ldE, cv);
}

template <int E>
static void gather_gate_bwd_launch(int dtype, const void* dx, const int32_t* idx,
                                   const int32_t* pos, const float* w, const float* dw,
                                   const float* logits, const void* wg, const void* dres, void* dA,
                                   float* dlogits, int T_, int M, int k, int ldE, cudaStream_t s) {
  if (dtype == DT_F32)
    gather_gate_bwd_launch_t<float, E>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, k, ldE, s);
  else
    gather_gate_bwd_launch_t<bf16, E>(dx, idx, pos, w, dw, logits, wg, dres, dA, dlogits, T_, M, k, ldE, s);
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
// dWg[m][e] (+)= Σ_t A[t][m]·dl[t][e]  ([M × T]·[T × E], HBM-bound on A).
// Part kernel: a CTA owns 4·blockDim.x columns × one token split; a thread keeps a
// 4-column × EB-expert register tile (one 8/16-byte load of A per token), dl of the split
// is broadcast from shared memory.  Reduce kernel: sums the splits in order
// (deterministic).
constexpr int GW_COLS = 4;  // columns per thread

template <typename T, int E>
__global__ void __launch_bounds__(256) gate_wgrad_part_kernel(const T* __restrict__ a, const float* __restrict__ dl,
                                                              float* __restrict__ part, int T_, int M, int TS) {
  constexpr int EB = E > 16 ? 16 : E;
  extern __shared__ float4 dls4[];  // [TS][E] floats
  const float* dls = reinterpret_cast<const float*>(dls4);
  FM_PDL_ENTRY();
  const int t0 = blockIdx.y * TS;
  const int nt = min(TS, T_ - t0);
  for (int i = threadIdx.x; i < nt * E; i += blockDim.x) reinterpret_cast<float*>(dls4)[i] = dl[(int64_t)t0 * E + i];
  __syncthreads();
  const int m = (blockIdx.x * blockDim.x + threadIdx.x) * GW_COLS;
  if (m >= M) return;
  float* dst = part + (int64_t)blockIdx.y * E * M + m;  // [split][E][M]
#pragma unroll 1
  for (int e0 = 0; e0 < E; e0 += EB) {
    float acc[GW_COLS][EB];
#pragma unroll
    for (int c = 0; c < GW_COLS; ++c)
#pragma unroll
      for (int j = 0; j < EB; ++j) acc[c][j] = 0.f;
#pragma unroll 4
    for (int t = 0; t < nt; ++t) {
      float x[GW_COLS];
      load_n<T, GW_COLS>(a + (int64_t)(t0 + t) * M + m, x);
      float d[EB];
      if constexpr (EB % 4 == 0) {
#pragma unroll
        for (int j = 0; j < EB; j += 4) {
          const float4 q = dls4[(t * E + e0 + j) >> 2];
          d[j] = q.x; d[j + 1] = q.y; d[j + 2] = q.z; d[j + 3] = q.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < EB; ++j) d[j] = dls[t * E + e0 + j];
      }
#pragma unroll
      for (int j = 0; j < EB; ++j)
#pragma unroll
        for (int c = 0; c < GW_COLS; ++c) acc[c][j] = fmaf(x[c], d[j], acc[c][j]);
    }
#pragma unroll
    for (int j = 0; j < EB; ++j) {
      float4 o;
      o.x = acc[0][j]; o.y = acc[1][j]; o.z = acc[2][j]; o.w = acc[3][j];
      *reinterpret_cast<float4*>(dst + (int64_t)(e0 + j) * M) = o;
    }
  }
}

// dwg[m][e] (+)= Σ_sp part[sp][e][m] in split order; thread = (e, m) with m fastest
__global__ void gate_wgrad_reduce_kernel(const float* __restrict__ part, float* __restrict__ dwg, int nsplit, int M,
                                         int E, int accumulate) {
  FM_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= M * E) return;
  const int e = i / M, m = i - e * M;
  float s = 0.f;
  for (int p = 0; p < nsplit; ++p) s += part[(int64_t)p * M * E + i];
  float* o = dwg + (int64_t)m * E + e;
  *o = accumulate ? *o + s : s;
}

// threads per CTA, token-split length and count: ~148 CTAs, splits of >= 16 tokens
static void gate_wgrad_geom(int T_, int M, int E, int* threads, int* TS, int* nsplit) {
  int th = (M / GW_COLS + 31) / 32 * 32;
  if (th > 256) th = 256;
  const int ctiles = (M / GW_COLS + th - 1) / th;
  int ns = (148 + ctiles - 1) / ctiles;
  const int max_ts = 4096 / E;  // dl tile <= 16 KB of shared memory
  int ts = (T_ + ns - 1) / ns;
  if (ts < 16) ts = 16;
  if (ts > max_ts) ts = max_ts;
  ns = (T_ + ts - 1) / ts;
  *threads = th; *TS = ts; *nsplit = ns;
}

size_t gate_wgrad_scratch_floats(int T_, int M, int E) {
  int th, ts, ns;
  gate_wgrad_geom(T_, M, E, &th, &ts, &ns);
  return (size_t)ns * M * E;
}

template <int E>
static void gate_wgrad_launch(int dtype, const void* a, const float* dl, float* part, int T_,
                              int M, cudaStream_t s) {
  int th, ts, ns;
  gate_wgrad_geom(T_, M, E, &th, &ts, &ns);
  dim3 grid((M / GW_COLS + th - 1) / th, ns);
  const size_t smem = (size_t)ts * E * sizeof(float);
  if (dtype == DT_F32)
    launch_k(gate_wgrad_part_kernel<float, E>, grid, th, smem, s, (const float*)a, dl, part, T_, M, ts);
  else
    launch_k(gate_wgrad_part_kernel<bf16, E>, grid, th, smem, s, (const bf16*)a, dl, part, T_, M, ts);
}

int gate_wgrad(int dtype, const void* a, const float* dlogits, float* dwg, float* part, int T_,
               int M, int E, int accumulate, cudaStream_t s) {
  if (T_ <= 0) return 0;
  FM_E_SWITCH(E, gate_wgrad_launch, dtype, a, dlogits, part, T_, M, s)
  int th, ts, ns;
  gate_wgrad_geom(T_, M, E, &th, &ts, &ns);
  launch_k(gate_wgrad_reduce_kernel, (M * E + 255) / 256, 256, 0, s, part, dwg, ns, M, E, accumulate);
  return (int)cudaGetLastError();
}

// ------------------------------------------------------------------ bias grads
// out[b][n] (+)= Σ_r x[b][r][n].  Block = 8 column-vector lanes × 32 row groups: a thread
// owns one 16-byte column vector and sums rows ry, ry+32, ...; the 32 partials are added
// in a fixed order (deterministic).  Narrow column tiles keep enough CTAs at small N.
template <typename T>
__global__ void __launch_bounds__(256) colsum_acc_kernel(const T* x, float* out, int rows, int N, int accumulate) {
  constexpr int V = 16 / sizeof(T);
  __shared__ float part[32][8 * V + 1];
  FM_PDL_ENTRY();
  const int cx = threadIdx.x & 7, ry = threadIdx.x >> 3;
  const int n0 = (blockIdx.x * 8 + cx) * V, b = blockIdx.y;
  const T* xb = x + (int64_t)b * rows * N;
  float s[V];
#pragma unroll
  for (int v = 0; v < V; ++v) s[v] = 0.f;
  if (n0 < N)
#pragma unroll 4
    for (int r = ry; r < rows; r += 32) {
      float v8[V];
      load16<T>(xb + (int64_t)r * N + n0, v8);
#pragma unroll
      for (int v = 0; v < V; ++v) s[v] += v8[v];
    }
#pragma unroll
  for (int v = 0; v < V; ++v) part[ry][cx * V + v] = s[v];
  __syncthreads();
  if (threadIdx.x < 8 * V) {
    const int n = blockIdx.x * 8 * V + threadIdx.x;
    if (n < N) {
      float t = 0.f;
#pragma unroll 8
      for (int i = 0; i < 32; ++i) t += part[i][threadIdx.x];
      out[(int64_t)b * N + n] = accumulate ? out[(int64_t)b * N + n] + t : t;
    }
  }
}

int colsum_acc(int dtype, const void* x, float* out, int batch, int rows, int N, int accumulate,
               cudaStream_t s) {
  const int V = dtype == DT_F32 ? 4 : 8;
  dim3 grid((N / V + 7) / 8, batch);
  if (dtype == DT_F32) launch_k(colsum_acc_kernel<float>, grid, 256, 0, s, (const float*)x, out, rows, N, accumulate);
  else launch_k(colsum_acc_kernel<bf16>, grid, 256, 0, s, (const bf16*)x, out, rows, N, accumulate);
  return (int)cudaGetLastError();
}

}  // namespace fm
