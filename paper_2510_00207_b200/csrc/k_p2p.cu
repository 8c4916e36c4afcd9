// A2A over NVLink peer memory: the dispatch / combine exchanges
// (S6, S8, B1, B3) as stores from this GPU's SMs straight into the peers' receive
// buffers (CUDA-IPC-mapped), completed by system-scope release counters.
//
// Protocol per (kind, chunk) use — no host involvement, CUDA-graph capturable:
//   sender  : CTAs copy 16-byte vectors of each C×M block to the destination rank's
//             buffer; each CTA fences (system scope) and bumps a local per-destination
//             piece counter; the CTA completing a destination fences again and atomically
//             increments that destination's arrival counter flags[kind][r][me] (remote
//             atomic over NVLink), then resets the piece counter.
//   receiver: one CTA waits (acquire loads) until flags[kind][r][src] >= seen + 1 for
//             every source, then seen += 1.  Counters are monotonic, so graph replays
//             and repeated blocks need no resets.  A spin bounded by ~10 s sets an error
//             word instead of hanging (checked by flowmoe_allreduce_wait).
#include "common.cuh"
#include "kernels.h"

namespace fm {

struct P2PArgs {
  const uint8_t* src;       // local source buffer (owner or expert side)
  uint8_t* dst[8];          // per-destination-rank receive buffer (mapped peer pointer or local)
  unsigned int* peer_flags[8];  // per-destination-rank arrival counters, indexed [kind][R][P]
  unsigned int* piece_cnt;  // local [kind][R][P] piece counters
  // fused wait (send_wait kernel): the grid's last CTA waits for every source
  const unsigned int* my_flags;  // my arrival counters [kind][R][P]
  unsigned int* seen;            // [kind][R] completed receives
  unsigned int* err;
  unsigned int* grid_cnt;        // [kind][R] CTA completion counter of the send grid
  int kind, r, R, P, El, me;
  int to_experts;           // 1: owner [E][R][C] -> expert [El][R][P][C]; 0: the reverse
  int64_t blk_bytes;        // C*M*es
  int pieces;               // CTAs per (destination, local expert) block
};

// A timed-out wait must not let its consumers read stale buffers (the arrival counters
// would then stay out of step with `seen` for good): flag it, then trap, which faults the
// context so the next stream synchronisation / flowmoe_check_health reports it.
FM_DEV void timeout_trap(unsigned int* err) {
  atomicExch(err, 1u);
  __threadfence_system();
  __trap();
}

// wait until every source published (kind, r) for the (seen + 1)-th time, then seen += 1
FM_DEV void p2p_wait_sources(const unsigned int* flags, unsigned int* seen, unsigned int* err, int kind, int r,
                             int R, int P) {
  const unsigned int expect = seen[kind * R + r] + 1u;
  const long long t0 = clock64();
  for (int q = 0; q < P; ++q) {
    const unsigned int* f = flags + ((int64_t)kind * R + r) * P + q;
    unsigned int v;
    while (true) {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if ((int)(v - expect) >= 0) break;
      if (clock64() - t0 > (1ll << 35)) {  // ~10-20 s: a peer is gone
        timeout_trap(err);
        break;
      }
      __nanosleep(32);
    }
  }
  seen[kind * R + r] = expect;
}

FM_DEV int64_t owner_off(int e, int r, int R, int64_t blk) { return ((int64_t)e * R + r) * blk; }
FM_DEV int64_t expert_off(int el, int r, int q, int R, int P, int64_t blk) {
  return (((int64_t)el * R + r) * P + q) * blk;
}

// one CTA's piece [v0, v1) of 16-byte words: 8 loads in flight per thread before the (remote)
// stores — a plain load->store loop keeps one load per thread outstanding and is bound by
// HBM latency, not by NVLink
FM_DEV void copy_piece(uint4* __restrict__ d, const uint4* __restrict__ s, int64_t v0, int64_t v1) {
  const int bd = blockDim.x;
  int64_t i = v0 + threadIdx.x;
  for (; i + 7 * bd < v1; i += 8 * bd) {
    uint4 t[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) t[j] = __ldg(s + i + j * bd);
#pragma unroll
    for (int j = 0; j < 8; ++j) d[i + j * bd] = t[j];
  }
  for (; i < v1; i += bd) d[i] = __ldg(s + i);
}

// grid (pieces, El, P): x = piece of the block, y = local expert, z = destination rank
__global__ void __launch_bounds__(256) a2a_p2p_send_kernel(P2PArgs a) {
  FM_PDL_ENTRY();
  const int piece = blockIdx.x, el = blockIdx.y, q = blockIdx.z;
  int64_t soff, doff;
  if (a.to_experts) {  // my owner-side block of expert (q, el) -> q's expert side slot (el, r, me)
    soff = owner_off(q * a.El + el, a.r, a.R, a.blk_bytes);
    doff = expert_off(el, a.r, a.me, a.R, a.P, a.blk_bytes);
  } else {  // my expert-side block (el, r, q) -> q's owner side slot (me*El + el, r)
    soff = expert_off(el, a.r, q, a.R, a.P, a.blk_bytes);
    doff = owner_off(a.me * a.El + el, a.r, a.R, a.blk_bytes);
  }
  const int64_t per = (a.blk_bytes / 16 + a.pieces - 1) / a.pieces;  // uint4 per piece
  const int64_t v0 = piece * per, v1 = min(a.blk_bytes / 16, v0 + per);
  const uint4* s = reinterpret_cast<const uint4*>(a.src + soff);
  uint4* d = reinterpret_cast<uint4*>(a.dst[q] + doff);
  copy_piece(d, s, v0, v1);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int* cnt = a.piece_cnt + ((int64_t)a.kind * a.R + a.r) * a.P + q;
    const unsigned int total = (unsigned int)(a.pieces * a.El);
    if (atomicAdd(cnt, 1u) == total - 1) {  // every piece for destination q has landed
      __threadfence_system();
      atomicAdd_system(a.peer_flags[q] + ((int64_t)a.kind * a.R + a.r) * a.P + a.me, 1u);
      *cnt = 0u;
    }
  }
}

// send + wait in one grid: every CTA copies its piece and publishes as in the send
// kernel; the CTA that completes the grid then waits for every source (one launch per
// exchange instead of two on the chunk's lane).
__global__ void __launch_bounds__(256) a2a_p2p_send_wait_kernel(P2PArgs a) {
  // No early trigger of the dependent launch: a consumer launched while this grid waits
  // for the peers could fill every SM (e.g. a persistent GEMM parked at its griddepcontrol
  // wait) and starve another lane's exchange that a peer is waiting on — a cross-rank
  // deadlock.  The completing CTA triggers it once every source has arrived.
  griddep_wait();
  __shared__ unsigned int last;
  const int piece = blockIdx.x, el = blockIdx.y, q = blockIdx.z;
  int64_t soff, doff;
  if (a.to_experts) {
    soff = owner_off(q * a.El + el, a.r, a.R, a.blk_bytes);
    doff = expert_off(el, a.r, a.me, a.R, a.P, a.blk_bytes);
  } else {
    soff = expert_off(el, a.r, q, a.R, a.P, a.blk_bytes);
    doff = owner_off(a.me * a.El + el, a.r, a.R, a.blk_bytes);
  }
  const int64_t per = (a.blk_bytes / 16 + a.pieces - 1) / a.pieces;
  const int64_t v0 = piece * per, v1 = min(a.blk_bytes / 16, v0 + per);
  const uint4* s = reinterpret_cast<const uint4*>(a.src + soff);
  uint4* d = reinterpret_cast<uint4*>(a.dst[q] + doff);
  copy_piece(d, s, v0, v1);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int* cnt = a.piece_cnt + ((int64_t)a.kind * a.R + a.r) * a.P + q;
    const unsigned int total = (unsigned int)(a.pieces * a.El);
    if (atomicAdd(cnt, 1u) == total - 1) {
      __threadfence_system();
      atomicAdd_system(a.peer_flags[q] + ((int64_t)a.kind * a.R + a.r) * a.P + a.me, 1u);
      *cnt = 0u;
    }
    unsigned int* gc = a.grid_cnt + a.kind * a.R + a.r;
    last = atomicAdd(gc, 1u) == gridDim.x * gridDim.y * gridDim.z - 1u;
    if (last) *gc = 0u;
  }
  __syncthreads();
  if (last) {
    if (threadIdx.x == 0) p2p_wait_sources(a.my_flags, a.seen, a.err, a.kind, a.r, a.R, a.P);
    __syncthreads();
    griddep_launch();
  }
}

// one CTA of P threads: wait for all sources of (kind, r)
__global__ void a2a_p2p_wait_kernel(const unsigned int* flags, unsigned int* seen, unsigned int* err,
                                    int kind, int r, int R, int P) {
  griddep_wait();  // dependents launch only when the wait is over (see the send+wait kernel)
  __shared__ unsigned int expect;
  if (threadIdx.x == 0) expect = seen[kind * R + r] + 1u;
  __syncthreads();
  const int q = threadIdx.x;
  if (q < P) {
    const unsigned int* f = flags + ((int64_t)kind * R + r) * P + q;
    const long long t0 = clock64();
    unsigned int v;
    do {
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
      if ((int)(v - expect) >= 0) break;
      if (clock64() - t0 > (1ll << 35)) {  // ~10-20 s: a peer is gone
        timeout_trap(err);
        break;
      }
      __nanosleep(64);
    } while (true);
  }
  __syncthreads();
  if (threadIdx.x == 0) seen[kind * R + r] = expect;
}

// Simulated world (flowmoe_create_local_group): sum of the P ranks' fp32 buffers over
// [off, off+n), in rank order, written back to every rank (one thread per element or
// 4-float vector: each reads all P values before writing, so in place is safe).
struct LocalArArgs {
  float* b[8];
  int P;
  int64_t off, n;
};

__global__ void __launch_bounds__(256) local_allreduce_kernel(LocalArArgs a) {
  FM_PDL_ENTRY();
  const int64_t nv = a.n / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int q = 0; q < a.P; ++q) {
      const float4 v = reinterpret_cast<const float4*>(a.b[q] + a.off)[i];
      acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
    }
    for (int q = 0; q < a.P; ++q) reinterpret_cast<float4*>(a.b[q] + a.off)[i] = acc;
  }
  for (int64_t i = nv * 4 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < a.n; i += stride) {
    float acc = 0.f;
    for (int q = 0; q < a.P; ++q) acc += a.b[q][a.off + i];
    for (int q = 0; q < a.P; ++q) a.b[q][a.off + i] = acc;
  }
}

int local_allreduce(float* const* bufs, int P, int64_t off, int64_t n, cudaStream_t s) {
  if (P > 8 || n < 0) return (int)cudaErrorInvalidValue;
  LocalArArgs a;
  for (int q = 0; q < 8; ++q) a.b[q] = q < P ? bufs[q] : nullptr;
  for (int q = 0; q < P; ++q)  // the vector path needs 16-byte aligned chunk starts
    if ((reinterpret_cast<uintptr_t>(bufs[q] + off) & 15) != 0) return (int)cudaErrorMisalignedAddress;
  a.P = P; a.off = off; a.n = n;
  const int64_t nv = (n + 3) / 4;
  int grid = (int)((nv + 255) / 256);
  grid = grid < 1 ? 1 : (grid > 4 * 148 ? 4 * 148 : grid);
  launch_k(local_allreduce_kernel, grid, 256, 0, s, a);
  return (int)cudaGetLastError();
}

int a2a_p2p(const void* src, void* const* dst, unsigned int* const* peer_flags, unsigned int* piece_cnt,
            unsigned int* my_flags, unsigned int* seen, unsigned int* err, int kind, int r, int R, int P,
            int El, int me, int to_experts, int64_t blk_bytes, cudaStream_t send_stream,
            cudaStream_t wait_stream, bool do_send, bool do_wait, unsigned int* grid_cnt) {
  if (P > 8) return (int)cudaErrorInvalidValue;
  if (do_send && do_wait && send_stream == wait_stream && grid_cnt) {  // one launch
    P2PArgs a;
    a.src = reinterpret_cast<const uint8_t*>(src);
    for (int q = 0; q < 8; ++q) {
      a.dst[q] = q < P ? reinterpret_cast<uint8_t*>(dst[q]) : nullptr;
      a.peer_flags[q] = q < P ? peer_flags[q] : nullptr;
    }
    a.piece_cnt = piece_cnt;
    a.my_flags = my_flags; a.seen = seen; a.err = err; a.grid_cnt = grid_cnt;
    a.kind = kind; a.r = r; a.R = R; a.P = P; a.El = El; a.me = me; a.to_experts = to_experts;
    a.blk_bytes = blk_bytes;
    a.pieces = (int)((blk_bytes + 32767) / 32768);
    launch_k(a2a_p2p_send_wait_kernel, dim3(a.pieces, El, P), 256, 0, send_stream, a);
    return (int)cudaGetLastError();
  }
  if (do_send) {
    P2PArgs a;
    a.src = reinterpret_cast<const uint8_t*>(src);
    for (int q = 0; q < 8; ++q) {
      a.dst[q] = q < P ? reinterpret_cast<uint8_t*>(dst[q]) : nullptr;
      a.peer_flags[q] = q < P ? peer_flags[q] : nullptr;
    }
    a.piece_cnt = piece_cnt;
    a.kind = kind; a.r = r; a.R = R; a.P = P; a.El = El; a.me = me; a.to_experts = to_experts;
    a.blk_bytes = blk_bytes;
    a.pieces = (int)((blk_bytes + 32767) / 32768);  // ~32 KB per CTA
    launch_k(a2a_p2p_send_kernel, dim3(a.pieces, El, P), 256, 0, send_stream, a);
    if (cudaError_t e = cudaGetLastError()) return (int)e;
  }
  if (do_wait) {
    launch_k(a2a_p2p_wait_kernel, 1, 32, 0, wait_stream, (const unsigned int*)my_flags, seen, err, kind, r, R, P);
  }
  return (int)cudaGetLastError();
}

}  // namespace fm
