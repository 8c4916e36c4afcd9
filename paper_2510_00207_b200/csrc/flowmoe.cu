// libflowmoe.so — C ABI + chunk scheduler of the FlowMoE block hot path.
//
// One ctx per rank (one process per GPU).  Three CUDA streams:
//   s_comp (compute tasks AT_r, E_r and their backward, in Eq.(3)/(5) order),
//   s_a2a  (highest priority: NCCL all-to-all D_r, C_r in Eq.(4)/(6) order),
//   s_ar   (lowest priority: chunked NCCL all-reduce of the MHA+gate grads).
// Dependencies between chunks are cudaEvents (the paper's DataQueue);
// the A2A and AR op orders are static and identical on every rank, so the two
// NCCL communicators never see diverging op orders (SURVEY.md §7 hard part 4).
// The AR chunks are released as soon as the grads they cover are final
// (reading Q10) and run on the low-priority stream/communicator, in
// the gaps left by the A2A stream (Alg. 2's "A2A first" rule).
#include <cuda_runtime.h>
#include <nccl.h>
#include <math.h>
#include <stdlib.h>
#include <stdio.h>
#include <string.h>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <mutex>
#include <string>
#include <map>
#include <vector>
#include <cuda.h>

#include "../../include/flowmoe.h"
#include "../../include/flowmoe_test.h"
#include "kernels.h"

using namespace fm;

namespace fm {
int g_pdl_enabled = 1;
// Peer-memory A2A of chunk r on chunk r's compute lane (1, default) or on the A2A
// stream of the NCCL path (0, debug key 6): with one lane per chunk the lane has
// nothing else to run while its chunk waits for the exchange, and staying on the lane
// saves two cross-stream event hops per exchange.
int g_p2p_on_lane = 1;
}

namespace {

thread_local std::string g_err;
std::atomic<uint64_t> g_launches{0};

flowmoe_status fail(flowmoe_status s, const std::string& msg) {
  g_err = msg;
  return s;
}

constexpr int NUM_TICKET_EVENTS = 4096;

struct SavedLayout {
  size_t qkv, ctx, lse, a, logits, idx, w, pos, counts, src, send, xe, z, h, ye, yc, dye, total;
};

// ---- per-kernel profiling (eager mode only; bench.py's live roofline) ----
enum KKind {
  KK_QKV, KK_ATTN_F, KK_OPROJ, KK_GATE, KK_ROUTE, KK_PACK, KK_E1, KK_E2, KK_COMBINE,
  KK_CBPACK, KK_DGELU, KK_DW2, KK_DB2, KK_DW1, KK_DB1, KK_DXE, KK_GATHER, KK_DCTX, KK_ATTN_B,
  KK_DX, KK_DWG, KK_DWO, KK_DWQKV, KK_A2A_D, KK_A2A_C, KK_A2A_CB, KK_A2A_DB, KK_AR, KK_TEST, KK_COUNT
};
const char* KK_NAMES[KK_COUNT] = {
  "gemm_qkv", "attn_fwd", "gemm_oproj", "gate_topk", "route_scan", "permute_pack",
  "gemm_expert1_gelu", "gemm_expert2", "unpermute_combine", "combine_bwd_pack", "gemm_expert_dgelu",
  "gemm_expert_dw2", "colsum_db2", "gemm_expert_dw1", "colsum_db1", "gemm_expert_dx",
  "gather_gate_bwd", "gemm_dctx", "attn_bwd", "gemm_dx", "gate_wgrad", "gemm_dwo", "gemm_dwqkv",
  "a2a_dispatch", "a2a_combine", "a2a_combine_bwd", "a2a_dispatch_bwd", "allreduce_chunk", "test_gemm"};
struct ProfRec { int kind; int ev; double flops, bytes; };
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<ProfRec> recs;
};
// the profile of the ctx whose call is being enqueued (apply_ctx); null = off
thread_local Prof* g_prof = nullptr;

// Task log (flowmoe_tasklog_*, flowmoe_test.h): each task of the schedule — AT_r, D_r, E_r,
// C_r, the merge, and backward C_r^bwd pack/exchange, E_r^bwd, D_r^bwd, AT_r^bwd, the
// weight-gradient tasks, every AR chunk — bracketed by timing events on its own stream,
// labelled (kind, block, chunk), so the Eq.(3)-(6) orders and the 6a-6e dependencies can be
// checked on measured timelines.  Eager enqueues only (not in capture).
enum TaskKind { TK_AT, TK_D, TK_E, TK_C, TK_MERGE, TK_CBPACK, TK_CB, TK_EB, TK_DB, TK_WGE, TK_ATB, TK_WGA, TK_AR };
struct TaskRec { int kind, block, chunk, dir; unsigned long long stream; int ev; };
struct TaskLog {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<TaskRec> recs;
  cudaEvent_t base = nullptr;
  int fwd_seq = 0, bwd_seq = 0, block = 0, dir = 0;
  std::mutex mu;  // simulated world: another member's thread records this rank's AR tasks
};

int prof_start(cudaStream_t s) {
  if (!g_prof || !g_prof->on) return -1;
  cudaStreamCaptureStatus cs;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return -1;
  Prof& pr = *g_prof;
  while (pr.pool.size() < pr.used + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    pr.pool.push_back(e);
  }
  int i = (int)pr.used;
  pr.used += 2;
  cudaEventRecord(pr.pool[i], s);
  return i;
}
void prof_stop(int i, int kind, double flops, double bytes, cudaStream_t s) {
  if (i < 0 || !g_prof) return;
  cudaEventRecord(g_prof->pool[i + 1], s);
  g_prof->recs.push_back({kind, i, flops, bytes});
}
#define FM_KP(kind, nk, fl, by, strm, call)            \
  do {                                                  \
    int pi_ = prof_start(strm);                         \
    FM_K(nk, call);                                     \
    prof_stop(pi_, kind, (double)(fl), (double)(by), strm); \
  } while (0)


size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

}  // namespace

struct LocalGroup;

struct flowmoe_ctx {
  flowmoe_config cfg;
  int dev = 0;
  int64_t T = 0, Tr = 0, S = 0, C = 0, El = 0, P = 1, F = 0, M = 0, E = 0, k = 1, H = 1, N = 1;
  size_t es = 2;
  int dt = DT_BF16;
  cudaStream_t s_comp = nullptr, s_a2a = nullptr, s_ar = nullptr;
  // compute lanes: lanes[0] == s_comp; chunk r's compute tasks run on lanes[r % n_lanes]
  std::vector<cudaStream_t> lanes;
  std::vector<cudaEvent_t> ev_lane;
  // stream-K GEMM scratch (k_gemm_tc.cu), one set per lane: lanes run GEMMs concurrently
  std::vector<float*> sk_ws;
  std::vector<unsigned int*> sk_tick;
  float* sk_test_ws = nullptr;  // flowmoe_test_gemm's (allocated on first use)
  unsigned int* sk_test_tick = nullptr;
  // per-block weight-grad stream (expert wgrads over all chunks, deferred MHA/gate
  // wgrads); == s_comp with one lane, its own stream with several
  cudaStream_t s_wg = nullptr;
  // A2A lanes (P > 1): chunk r's A2As use a2a_comm[r % n] on a2a_stream[r % n]
  // (index 0 = comm_a2a / s_a2a); each communicator sees a static op order.
  std::vector<ncclComm_t> a2a_comm;
  std::vector<cudaStream_t> a2a_stream;
  ncclComm_t comm_a2a = nullptr, comm_ar = nullptr;
  // per-chunk events
  std::vector<cudaEvent_t> ev_at, ev_d, ev_e, ev_c, ev_cb, ev_cba, ev_eb, ev_dba;
  // token chunks (chunk = causal slice of one sequence, reading Q1'): chunk r's attention
  // reads Q/K/V of the earlier chunks of its sequence (ev_qkv) and, backward, the dctx
  // of the later ones (ev_dctx); a chunk's dctx rows may be rewritten by the next
  // block's backward only after the earlier chunks' attention backward read them (ev_atb)
  bool tok = false;
  std::vector<cudaEvent_t> ev_qkv, ev_dctx, ev_atb;
  std::vector<unsigned long long> atb_cap;  // capture id at record time
  std::vector<char> atb_rec;
  cudaEvent_t ev_in = nullptr, ev_done = nullptr, ev_grads_a = nullptr, ev_grads_b = nullptr;
  cudaEvent_t ev_bwd_done = nullptr;  // end of the latest block_bwd (centralized AR starts after it)
  std::vector<cudaEvent_t> ticket_ev;
  uint64_t next_ticket = 1;
  SavedLayout L{};
  // backward workspaces (ctx-owned, reused by every block)
  void *dyc = nullptr, *dye = nullptr, *dz = nullptr, *dxe = nullptr, *dxc = nullptr;
  // workspaces read by the weight-grad stream come in two sets when that stream is
  // separate, so block l's wgrads overlap block l-1's backward (set = call parity)
  void *ws_dyc[2] = {}, *ws_dye[2] = {}, *ws_dz[2] = {}, *ws_dA[2] = {}, *ws_dqkv[2] = {};
  float* ws_dl[2] = {};
  cudaEvent_t ev_wg_done[2] = {};
  unsigned long long wg_cap_id[2] = {};  // capture id at record time (0 = eager)
  bool wg_recorded[2] = {false, false};
  uint64_t bwd_calls = 0;
  void *dA = nullptr, *dctx = nullptr, *dqkv = nullptr;
  float *dl = nullptr, *dw = nullptr, *Dbuf = nullptr, *wg_part = nullptr;
  unsigned int* route_done = nullptr;  // [R] last-CTA counters of the fused gate+route kernel
  std::vector<void*> allocs;
  const int32_t* forced = nullptr;
  // ---- A2A over NVLink peer memory (a2a_impl = FLOWMOE_A2A_P2P)
  bool p2p = false;
  void* p2p_arena = nullptr;            // [flags 4*R*P | piece counters 4*R*P | seen 4*R | err]
  unsigned int *flags = nullptr, *piece_cnt = nullptr, *seen = nullptr, *p2p_err = nullptr;
  unsigned int* grid_cnt = nullptr;      // [4*R] CTA counters of the fused send+wait kernel
  std::vector<unsigned int*> peer_flags; // per rank: its flags array (mapped)
  std::vector<void*> peer_dxc;           // per rank: its dispatch-bwd receive buffer (mapped)
  std::map<const void*, std::vector<void*>> peer_saved;  // my saved ptr -> each rank's saved ptr
  std::map<const void*, std::vector<void*>> saved_opened;  // my saved ptr -> peer mappings opened for it
  std::vector<void*> ipc_opened;         // peer mappings to close at destroy
  void* xchg = nullptr;                  // device scratch of the registration collectives
  // scheduling policy (flowmoe_schedule): AT split into R subtasks? AR chunked per block?
  bool at_split = true, ar_pipelined = true;
  struct PendingAR { float* buf; size_t count; uint64_t ticket; };
  std::vector<PendingAR> pending_ar;  // centralized-AR policies: flushed at allreduce_wait
  // per-ctx test/benchmark knobs (flowmoe_test.h) and per-kernel profile, applied to the
  // kernel modules by apply_ctx() at the start of every enqueueing call
  int dbg_flags = 0, pdl = 1, force_bn = 0, force_cg = 0, force_sk = 0, p2p_on_lane = 1;
  // SMs the backward GEMMs leave to the all-reduce at P > 1 (the AR communicator's CTA cap
  // on a real multi-GPU ctx; key 9 overrides, 0 = none) and the cap of the GEMMs being enqueued
  int bwd_sm_reserve = 0, gemm_max_sms = 0;
  int sm_reserve = 0;  // key 10: SMs every GEMM leaves to the other lanes' kernels (A/B; 0 = none)
  Prof prof;
  TaskLog tlog;
  // saved stashes registered for peer-memory A2A, in registration order (collective)
  std::vector<const void*> saved_order;
  // in-process simulated world (flowmoe_create_local_group): P ctxs on one device
  LocalGroup* group = nullptr;
  std::vector<cudaEvent_t> ev_sent;  // simulated world: [4 kinds][R] end of this rank's send
};

// In-process simulated world (flowmoe_create_local_group, include/flowmoe_test.h): P ctxs
// of world_size P on ONE device, so the exchange rows (S6, S8, B1, B3: the peer-memory A2A
// kernels and their arrival counters; B6: the S_p chunk loop of the all-reduce) run on a
// one-GPU box.  Peers' buffers are plain device pointers.  The all-reduce of a submission
// is enqueued once every rank has made its matching submission: it sums the P ranks'
// buffers chunk by chunk (same S_p partition as the NCCL path) in rank order on the
// group's stream and writes the sum back to every rank.
struct LocalGroup {
  int P = 0;
  std::vector<flowmoe_ctx*> m;                   // members by rank (null once destroyed)
  std::vector<std::vector<const void*>> saved;   // registered stashes per rank, in order
  cudaStream_t s = nullptr;
  struct Sub { float* buf; size_t count, chunk_bytes; cudaEvent_t ready; int block; };
  std::vector<std::vector<Sub>> subs;            // per rank, AR submissions in order
  std::vector<std::map<uint64_t, size_t>> ticket_sub;  // per rank: ticket -> its last submission
  std::vector<std::map<uint64_t, size_t>> ticket_done;  // per rank: enqueued tickets
  size_t done = 0;                               // submissions enqueued (same index on every rank)
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  // member threads: barrier of the exchanges, lock of the shared state above
  std::mutex mu;
  std::condition_variable cv;
  int bar_count = 0;
  uint64_t bar_gen = 0;
};

namespace {

#define FM_CUDA(call)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (call);                                                               \
    if (e_ != cudaSuccess)                                                                 \
      return fail(FLOWMOE_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)
#define FM_NCCL(call)                                                                      \
  do {                                                                                     \
    ncclResult_t r_ = (call);                                                              \
    if (r_ != ncclSuccess)                                                                 \
      return fail(FLOWMOE_ERR_NCCL, std::string(#call) + ": " + ncclGetErrorString(r_));  \
  } while (0)
#define FM_K(nk, call)                                                                     \
  do {                                                                                     \
    int e_ = (call);                                                                       \
    g_launches += (nk);                                                                    \
    if (e_ != 0)                                                                           \
      return fail(FLOWMOE_ERR_CUDA, std::string(#call) + ": " +                            \
                                        cudaGetErrorString((cudaError_t)e_));              \
  } while (0)

// Install the ctx's knobs and profile into the (process-global) kernel modules for the
// call being enqueued; every enqueueing entry point calls this first.
void apply_ctx(flowmoe_ctx* x) {
  if (!x) return;
  gemm_tc_set_debug(x->dbg_flags);
  gemm_tc_force_bn(x->force_bn);
  gemm_tc_force_cg(x->force_cg);
  gemm_tc_force_streamk(x->force_sk);
  g_pdl_enabled = x->pdl;
  g_p2p_on_lane = x->p2p_on_lane;
  g_prof = &x->prof;
}

unsigned long long capture_id(cudaStream_t s);

int task_begin(flowmoe_ctx* x, cudaStream_t s) {
  TaskLog& tl = x->tlog;
  if (!tl.on || capture_id(s)) return -1;
  std::lock_guard<std::mutex> lk(tl.mu);
  while (tl.pool.size() < tl.used + 2) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return -1;
    tl.pool.push_back(e);
  }
  const int i = (int)tl.used;
  tl.used += 2;
  cudaEventRecord(tl.pool[i], s);
  return i;
}
void task_end(flowmoe_ctx* x, int i, int kind, int chunk, cudaStream_t s, int block = -1) {
  if (i < 0) return;
  TaskLog& tl = x->tlog;
  std::lock_guard<std::mutex> lk(tl.mu);
  cudaEventRecord(tl.pool[i + 1], s);
  unsigned long long sid = 0;
  cudaStreamGetId(s, &sid);
  tl.recs.push_back({kind, block >= 0 ? block : tl.block, chunk, tl.dir, sid, i});
}

// GEMM with its algorithmic work: 2·M·N·K flops; bytes = A + B + C (+C read for fp32 accumulate)
flowmoe_status run_gemm(int kind, const GemmArgs& g, int dt, size_t es, cudaStream_t s) {
  const double b = g.batch;
  const double flops = 2.0 * g.M * g.N * (double)g.K * b;
  double bytes = ((double)g.M * g.K + (double)g.K * g.N) * es * b;
  bytes += g.epi == EPI_ACC_F32 ? 8.0 * g.M * g.N * b
                                 : (double)g.M * g.N * (g.epi == EPI_STORE_F32 ? 4 : es) * b;
  if (g.epi == EPI_BIAS_GELU || g.epi == EPI_DGELU || g.epi == EPI_BIAS_GELU_G || g.epi == EPI_MUL_AUX)
    bytes += (double)g.M * g.N * es * b;
  if (g.resid) bytes += (double)g.M * g.N * es * b;
  FM_KP(kind, 1, flops, bytes, s, gemm(g, dt, s));
  return FLOWMOE_OK;
}
// stream-K scratch: one fp32 partial tile (128 x 256) per CTA of a full grid, and counters
constexpr size_t SK_WS_FLOATS = (size_t)148 * 128 * 256;
constexpr size_t SK_TICKS = 1 << 16;
void set_streamk(const flowmoe_ctx* x, GemmArgs& g, cudaStream_t s) {
  for (size_t i = 0; i < x->sk_ws.size() && i < x->lanes.size(); ++i)
    if (x->lanes[i] == s) {
      g.splitk_ws = x->sk_ws[i]; g.splitk_ws_floats = SK_WS_FLOATS;
      g.splitk_tick = x->sk_tick[i]; g.splitk_ticks = SK_TICKS;
    }
}
#define FM_GEMM(kind, g)                                                   \
  do {                                                                     \
    set_streamk(x, g, sc);                                                 \
    g.max_sms = x->gemm_max_sms;                                           \
    if (flowmoe_status st_ = run_gemm(kind, g, dt, es, sc)) return st_;   \
  } while (0)

flowmoe_status validate(const flowmoe_config* c) {
  if (!c) return fail(FLOWMOE_ERR_INVALID, "config is NULL");
  auto bad = [](const char* f, const std::string& why) {
    return fail(FLOWMOE_ERR_INVALID, std::string("config.") + f + ": " + why);
  };
  if (c->B <= 0) return bad("B", "must be > 0");
  if (c->seq_len <= 0) return bad("seq_len", "must be > 0");
  if (c->B % c->seq_len) return bad("B", "must be a multiple of seq_len (whole sequences)");
  if (c->R <= 0) return bad("R", "must be >= 1");
  if (c->B % c->R) return bad("R", "must divide B (chunks of B/R tokens)");
  {
    const int64_t Tr = c->B / c->R;
    if (Tr % c->seq_len && (c->seq_len % Tr || !c->causal))
      return bad("R", "chunks of B/R tokens must be whole sequences (reading Q1) or, with causal = 1, "
                      "slices of one sequence (B/R dividing seq_len, reading Q1')");
  }
  if (c->M <= 0 || c->M % 8) return bad("M", "must be a positive multiple of 8");
  if (c->n_heads <= 0 || c->M % c->n_heads) return bad("n_heads", "must divide M");
  int dh = c->M / c->n_heads;
  if (dh != 16 && dh != 32 && dh != 64 && dh != 128) return bad("n_heads", "d_h = M/n_heads must be 16, 32, 64 or 128");
  if (c->E != 2 && c->E != 4 && c->E != 8 && c->E != 16 && c->E != 32 && c->E != 64)
    return bad("E", "must be one of 2,4,8,16,32,64");
  if (c->top_k < 1 || c->top_k > c->E || c->top_k > 8) return bad("top_k", "need 1 <= k <= min(E, 8)");
  if (c->d_ffn <= 0 || c->d_ffn % 8) return bad("d_ffn", "must be a positive multiple of 8");
  if (!(c->capacity_factor >= 0.f)) return bad("capacity_factor", "must be >= 0");
  if (c->causal != 0 && c->causal != 1) return bad("causal", "must be 0 or 1");
  if (c->residual != 0 && c->residual != 1) return bad("residual", "must be 0 or 1");
  if (c->dtype != FLOWMOE_F32 && c->dtype != FLOWMOE_BF16) return bad("dtype", "must be FLOWMOE_F32 or FLOWMOE_BF16");
  if (c->grad_mode != FLOWMOE_GRAD_ACCUMULATE && c->grad_mode != FLOWMOE_GRAD_OVERWRITE)
    return bad("grad_mode", "must be FLOWMOE_GRAD_ACCUMULATE or FLOWMOE_GRAD_OVERWRITE");
  if (c->schedule < FLOWMOE_SCHED_FLOWMOE || c->schedule > FLOWMOE_SCHED_VANILLA_EP)
    return bad("schedule", "must be a flowmoe_schedule value");
  if (c->a2a_impl != FLOWMOE_A2A_NCCL && c->a2a_impl != FLOWMOE_A2A_P2P)
    return bad("a2a_impl", "must be FLOWMOE_A2A_NCCL or FLOWMOE_A2A_P2P");
  if (c->a2a_impl == FLOWMOE_A2A_P2P && c->world_size > 8)
    return bad("a2a_impl", "peer-memory A2A supports world_size <= 8 (one NVLink domain)");
  if (c->compute_streams < 0) return bad("compute_streams", "must be >= 0 (0 or 1 = one compute stream)");
  if (c->world_size < 1) return bad("world_size", "must be >= 1");
  if (c->rank < 0 || c->rank >= c->world_size) return bad("rank", "must be in [0, world_size)");
  if (c->E % c->world_size) return bad("E", "must be a multiple of world_size (experts sharded evenly)");
  return FLOWMOE_OK;
}

int64_t capacity_of(const flowmoe_config* c, int64_t Tr) {
  // C = f·k·B·N/E, ceil; f = 0 => dropless (reading Q3)
  if (c->capacity_factor == 0.f) return Tr;
  return (int64_t)ceil((double)c->capacity_factor * (double)c->top_k * (double)Tr / (double)c->E);
}

SavedLayout layout_of(const flowmoe_ctx* x) {
  SavedLayout L{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off = align_up(off + bytes, 256);
    return o;
  };
  const size_t es = x->es;
  const int64_t T = x->T, M = x->M, E = x->E, k = x->k, R = x->cfg.R, C = x->C, F = x->F;
  L.qkv = take(T * 3 * M * es);
  L.ctx = take(T * M * es);
  L.lse = take(T * x->H * 4);
  L.a = take(T * M * es);
  L.logits = take(T * E * 4);
  L.idx = take(T * k * 4);
  L.w = take(T * k * 4);
  L.pos = take(T * k * 4);
  L.counts = take(R * E * 4);
  L.src = take(R * E * C * 4);
  L.send = take(R * E * C * M * es);
  L.xe = x->P > 1 ? take(R * E * C * M * es) : L.send;
  L.z = take(R * E * C * F * es);  // GELU'(Z), [El][R][P*C][F] == R*E*C*F elements
  L.h = take(R * E * C * F * es);
  L.ye = take(R * E * C * M * es);
  L.yc = x->P > 1 ? take(R * E * C * M * es) : L.ye;
  // P > 1: receive buffer of the backward combine A2A (dY on the expert side), per block so
  // that peers writing block l-1's dY can never race the wgrads still reading block l's
  L.dye = x->P > 1 ? take(R * E * C * M * es) : 0;
  L.total = off;
  return L;
}

ncclDataType_t nccl_dt(const flowmoe_ctx* x) { return x->dt == DT_BF16 ? ncclBfloat16 : ncclFloat; }

// Expert buffers are expert-major, chunk-minor so that one expert's rows over all
// R chunks are contiguous (the expert wgrads then run as ONE K = R·P·C GEMM):
//   owner side  [E][R][C][M]      (dispatch send, combine recv)
//   expert side [E/P][R][P][C][M] (dispatch recv, expert GEMM rows, combine send)
// Chunk r, destination/source rank q, local expert el: one C×M block each.
size_t owner_blk(const flowmoe_ctx* x, int64_t e, int r) { return (size_t)(e * x->cfg.R + r) * x->C * x->M; }
size_t expert_blk(const flowmoe_ctx* x, int64_t el, int r, int q) {
  return (size_t)((el * x->cfg.R + r) * x->P + q) * x->C * x->M;
}

// owner side -> expert side for chunk r (dispatch D_r, and C_r^bwd of dY)
flowmoe_status a2a_to_experts(flowmoe_ctx* x, const void* send, void* recv, int r) {
  const size_t blk = (size_t)x->C * x->M;
  const int ln = r % (int)x->a2a_comm.size();
  ncclComm_t comm = x->a2a_comm[ln];
  cudaStream_t st = x->a2a_stream[ln];
  FM_NCCL(ncclGroupStart());
  for (int q = 0; q < x->P; ++q)
    for (int el = 0; el < x->El; ++el) {
      FM_NCCL(ncclSend((const char*)send + owner_blk(x, q * x->El + el, r) * x->es, blk, nccl_dt(x), q,
                       comm, st));
      FM_NCCL(ncclRecv((char*)recv + expert_blk(x, el, r, q) * x->es, blk, nccl_dt(x), q,
                       comm, st));
    }
  FM_NCCL(ncclGroupEnd());
  return FLOWMOE_OK;
}

// expert side -> owner side for chunk r (combine C_r, and D_r^bwd of dX)
flowmoe_status a2a_to_owners(flowmoe_ctx* x, const void* send, void* recv, int r) {
  const size_t blk = (size_t)x->C * x->M;
  const int ln = r % (int)x->a2a_comm.size();
  ncclComm_t comm = x->a2a_comm[ln];
  cudaStream_t st = x->a2a_stream[ln];
  FM_NCCL(ncclGroupStart());
  for (int q = 0; q < x->P; ++q)
    for (int el = 0; el < x->El; ++el) {
      FM_NCCL(ncclSend((const char*)send + expert_blk(x, el, r, q) * x->es, blk, nccl_dt(x), q,
                       comm, st));
      FM_NCCL(ncclRecv((char*)recv + owner_blk(x, q * x->El + el, r) * x->es, blk, nccl_dt(x), q,
                       comm, st));
    }
  FM_NCCL(ncclGroupEnd());
  return FLOWMOE_OK;
}

// fork: every compute lane waits for the caller's stream
unsigned long long capture_id(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  unsigned long long id = 0;
  if (cudaStreamGetCaptureInfo(s, &st, &id) != cudaSuccess || st != cudaStreamCaptureStatusActive) return 0;
  return id;
}

flowmoe_status fork_lanes(flowmoe_ctx* x, cudaStream_t stream) {
  FM_CUDA(cudaEventRecord(x->ev_in, stream));
  for (cudaStream_t l : x->lanes) FM_CUDA(cudaStreamWaitEvent(l, x->ev_in, 0));
  return FLOWMOE_OK;
}
// join: `dst` waits for every compute lane other than itself
flowmoe_status join_lanes(flowmoe_ctx* x, cudaStream_t dst) {
  for (size_t l = 0; l < x->lanes.size(); ++l) {
    if (x->lanes[l] == dst) continue;
    FM_CUDA(cudaEventRecord(x->ev_lane[l], x->lanes[l]));
    FM_CUDA(cudaStreamWaitEvent(dst, x->ev_lane[l], 0));
  }
  return FLOWMOE_OK;
}

// broadcast: every other compute lane waits for the work enqueued so far on `src`
flowmoe_status lanes_follow(flowmoe_ctx* x, cudaStream_t src) {
  FM_CUDA(cudaEventRecord(x->ev_in, src));
  for (cudaStream_t l : x->lanes)
    if (l != src) FM_CUDA(cudaStreamWaitEvent(l, x->ev_in, 0));
  return FLOWMOE_OK;
}

// ---- CUDA-IPC exchange over the A2A communicator (outside graph capture only)
typedef CUresult (*PFN_getAddressRange)(CUdeviceptr*, size_t*, CUdeviceptr);

struct IpcRec {
  cudaIpcMemHandle_t h;
  uint64_t offset;
  int32_t ok;  // 0: this rank could not export the allocation (every rank then fails)
};

// every rank publishes (handle of the allocation containing `ptr`, offset of ptr in it);
// returns each rank's view pointer (own = ptr).  Collective over the A2A communicator and
// all-or-nothing: a rank that cannot export or open a handle still takes part in both
// agreement rounds, so either every rank maps every peer or every rank reports failure
// (and all of them fall back to NCCL together) — no rank is left waiting in a collective.
flowmoe_status ipc_exchange(flowmoe_ctx* x, void* ptr, std::vector<void*>* out, std::vector<void*>* opened_out) {
  static PFN_getAddressRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) == cudaSuccess && fn)
      get_range = reinterpret_cast<PFN_getAddressRange>(fn);
  }
  // quiesce: earlier NCCL work of this communicator (any stream) must be done on every
  // rank before the exchange collective (eager path, once per registered buffer)
  FM_CUDA(cudaDeviceSynchronize());
  IpcRec mine;
  memset(&mine, 0, sizeof(mine));
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range && get_range(&base, &size, (CUdeviceptr)ptr) == CUDA_SUCCESS &&
      cudaIpcGetMemHandle(&mine.h, reinterpret_cast<void*>(base)) == cudaSuccess) {
    mine.offset = (uint64_t)((CUdeviceptr)ptr - base);
    mine.ok = 1;
  }
  cudaGetLastError();  // a failed export is reported through the agreement, not here
  const int P = (int)x->P;
  IpcRec* d = reinterpret_cast<IpcRec*>(x->xchg);
  FM_CUDA(cudaMemcpy(d + P, &mine, sizeof(IpcRec), cudaMemcpyHostToDevice));
  FM_NCCL(ncclAllGather(d + P, d, sizeof(IpcRec), ncclUint8, x->comm_a2a, x->s_comp));
  FM_CUDA(cudaStreamSynchronize(x->s_comp));
  std::vector<IpcRec> all(P);
  FM_CUDA(cudaMemcpy(all.data(), d, sizeof(IpcRec) * P, cudaMemcpyDeviceToHost));
  bool ok = true;
  for (const IpcRec& r : all) ok = ok && r.ok;
  std::vector<void*> opened;
  out->assign(P, nullptr);
  for (int q = 0; q < P && ok; ++q) {
    if (q == x->cfg.rank) { (*out)[q] = ptr; continue; }
    void* pb = nullptr;
    if (cudaIpcOpenMemHandle(&pb, all[q].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      break;
    }
    opened.push_back(pb);
    (*out)[q] = reinterpret_cast<char*>(pb) + all[q].offset;
  }
  // second round: did every rank open every peer?
  int32_t* flag = reinterpret_cast<int32_t*>(d + P + 1);
  const int32_t mine_ok = ok ? 1 : 0;
  FM_CUDA(cudaMemcpy(flag, &mine_ok, sizeof(int32_t), cudaMemcpyHostToDevice));
  FM_NCCL(ncclAllReduce(flag, flag, 1, ncclInt32, ncclMin, x->comm_a2a, x->s_comp));
  FM_CUDA(cudaStreamSynchronize(x->s_comp));
  int32_t all_ok = 0;
  FM_CUDA(cudaMemcpy(&all_ok, flag, sizeof(int32_t), cudaMemcpyDeviceToHost));
  if (!all_ok) {
    for (void* pb : opened) cudaIpcCloseMemHandle(pb);
    out->clear();
    return fail(FLOWMOE_ERR_CUDA, "peer-memory registration failed on some rank (CUDA IPC export/open)");
  }
  for (void* pb : opened) opened_out->push_back(pb);
  return FLOWMOE_OK;
}

flowmoe_status register_saved(flowmoe_ctx* x, const void* saved);
flowmoe_status p2p_exchange(flowmoe_ctx* x, int kind, int r, const void* src, void* const* dst, int to_experts,
                            cudaStream_t sa);

// Peer-memory A2A for this `saved` stash?  *use = true when every rank's stash is mapped.
// A stash that was not registered (flowmoe_register_saved) is registered here on first
// sight, collectively, outside graph capture; during capture it uses NCCL (every rank sees
// the same sequence of calls, so every rank decides the same).  The in-process simulated
// world has no NCCL: there every stash must be registered on all ranks first.
flowmoe_status resolve_p2p(flowmoe_ctx* x, const void* saved, cudaStream_t stream, bool* use) {
  *use = false;
  if (x->P == 1 || !x->p2p) return FLOWMOE_OK;
  if (x->peer_saved.count(saved)) { *use = true; return FLOWMOE_OK; }
  if (!x->group) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(stream, &cs);
    if (cs != cudaStreamCaptureStatusNone) return FLOWMOE_OK;
    if (register_saved(x, saved) != FLOWMOE_OK) return FLOWMOE_OK;  // all ranks failed: NCCL
    *use = x->peer_saved.count(saved) > 0;
    return FLOWMOE_OK;
  }
  if (flowmoe_status st = register_saved(x, saved)) return st;
  {
    std::lock_guard<std::mutex> lk(x->group->mu);
    *use = x->peer_saved.count(saved) > 0;
  }
  if (!*use)
    return fail(FLOWMOE_ERR_STATE, "local group: saved stash not registered on every rank "
                                   "(call flowmoe_register_saved on each rank before the first block_fwd)");
  return FLOWMOE_OK;
}

template <typename P_>
P_* at(void* base, size_t off) { return reinterpret_cast<P_*>(reinterpret_cast<char*>(base) + off); }
template <typename P_>
const P_* at(const void* base, size_t off) {
  return reinterpret_cast<const P_*>(reinterpret_cast<const char*>(base) + off);
}

// The S_p partition of Alg. 2 PARTITION: chunks of chunk_bytes/4 floats, the
// last one the remainder.  Shared by the NCCL path and the simulated world.
template <typename F_>
flowmoe_status for_each_ar_chunk(size_t count, size_t chunk_bytes, F_&& f) {
  const size_t chunk = chunk_bytes / 4;
  for (size_t off = 0; off < count; off += chunk) {
    const size_t n = (count - off < chunk) ? count - off : chunk;
    if (flowmoe_status st = f(off, n)) return st;
  }
  return FLOWMOE_OK;
}

// simulated world: enqueue every submission index that all ranks have reached
flowmoe_status group_flush(LocalGroup* g) {
  while (true) {
    for (int q = 0; q < g->P; ++q)
      if (g->subs[q].size() <= g->done) return FLOWMOE_OK;
    const size_t n = g->done;
    const LocalGroup::Sub& s0 = g->subs[0][n];
    float* bufs[8] = {};
    for (int q = 0; q < g->P; ++q) {
      const LocalGroup::Sub& sq = g->subs[q][n];
      if (sq.count != s0.count || sq.chunk_bytes != s0.chunk_bytes)
        return fail(FLOWMOE_ERR_STATE, "local group: all-reduce submissions differ across ranks");
      FM_CUDA(cudaStreamWaitEvent(g->s, sq.ready, 0));
      bufs[q] = sq.buf;
    }
    int ci = 0;
    if (flowmoe_status st = for_each_ar_chunk(s0.count, s0.chunk_bytes, [&](size_t off, size_t cnt) {
          int tk[8];
          for (int q = 0; q < g->P; ++q) tk[q] = task_begin(g->m[q], g->s);
          int pi = prof_start(g->s);
          FM_K(1, local_allreduce(bufs, g->P, (int64_t)off, (int64_t)cnt, g->s));
          prof_stop(pi, KK_AR, 0, 4.0 * cnt * 2.0 * (g->P - 1) / g->P, g->s);
          for (int q = 0; q < g->P; ++q) task_end(g->m[q], tk[q], TK_AR, ci, g->s, g->subs[q][n].block);
          ++ci;
          return FLOWMOE_OK;
        }))
      return st;
    for (int q = 0; q < g->P; ++q)
      for (auto& kv : g->ticket_sub[q])
        if (kv.second == n) {
          FM_CUDA(cudaEventRecord(g->m[q]->ticket_ev[kv.first % NUM_TICKET_EVENTS], g->s));
          g->ticket_done[q][kv.first] = n;
        }
    g->done = n + 1;
  }
}

flowmoe_status submit_ar(flowmoe_ctx* x, float* buf, size_t count, size_t chunk_bytes,
                         cudaEvent_t ready) {
  if (ready) FM_CUDA(cudaStreamWaitEvent(x->s_ar, ready, 0));
  if (x->P == 1 || count == 0) return FLOWMOE_OK;
  if (LocalGroup* g = x->group) {
    std::lock_guard<std::mutex> lk(g->mu);
    // snapshot the readiness (the caller's event may be re-recorded by the next block)
    if (g->ev_used == g->ev_pool.size()) {
      cudaEvent_t e;
      FM_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      g->ev_pool.push_back(e);
    }
    cudaEvent_t e = g->ev_pool[g->ev_used++];
    FM_CUDA(cudaEventRecord(e, x->s_ar));
    g->subs[x->cfg.rank].push_back({buf, count, chunk_bytes, e, x->tlog.block});
    return group_flush(g);
  }
  int ci = 0;
  return for_each_ar_chunk(count, chunk_bytes, [&](size_t off, size_t n) {
    const int tk = task_begin(x, x->s_ar);
    int pi = prof_start(x->s_ar);
    FM_NCCL(ncclAllReduce(buf + off, buf + off, n, ncclFloat, ncclSum, x->comm_ar, x->s_ar));
    prof_stop(pi, KK_AR, 0, 4.0 * n * 2.0 * (x->P - 1) / x->P, x->s_ar);
    task_end(x, tk, TK_AR, ci++, x->s_ar);
    return FLOWMOE_OK;
  });
}

flowmoe_status new_ticket(flowmoe_ctx* x, flowmoe_ticket* out) {
  const uint64_t t = x->next_ticket++;
  LocalGroup* g = x->group;
  const int rk = x->cfg.rank;
  std::unique_lock<std::mutex> lk;
  if (g) lk = std::unique_lock<std::mutex>(g->mu);
  if (g && !g->subs[rk].empty() && g->subs[rk].size() > g->done) {
    g->ticket_sub[rk][t] = g->subs[rk].size() - 1;  // recorded when that submission is enqueued
  } else {
    // simulated world: this rank's all-reduces so far are on the group's stream
    FM_CUDA(cudaEventRecord(x->ticket_ev[t % NUM_TICKET_EVENTS], g ? g->s : x->s_ar));
  }
  if (out) *out = t;
  return FLOWMOE_OK;
}

}  // namespace

extern "C" {

const char* flowmoe_status_string(flowmoe_status s) {
  switch (s) {
    case FLOWMOE_OK: return "ok";
    case FLOWMOE_ERR_INVALID: return "invalid argument";
    case FLOWMOE_ERR_CUDA: return "CUDA error";
    case FLOWMOE_ERR_NCCL: return "NCCL error";
    case FLOWMOE_ERR_OOM: return "out of device memory";
    case FLOWMOE_ERR_UNSUPPORTED: return "unsupported";
    case FLOWMOE_ERR_STATE: return "invalid state";
  }
  return "unknown status";
}

const char* flowmoe_last_error(void) { return g_err.c_str(); }

uint64_t flowmoe_kernel_launches(void) { return g_launches.load(); }

flowmoe_status flowmoe_debug_set(flowmoe_ctx* x, int key, int value) {
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (key == 1) x->dbg_flags = (x->dbg_flags & ~1) | (value ? 1 : 0);
  else if (key == 2) x->dbg_flags = (x->dbg_flags & ~2) | (value ? 2 : 0);
  else if (key == 3) x->dbg_flags = (x->dbg_flags & ~4) | (value ? 4 : 0);
  else if (key == 4) x->pdl = value ? 1 : 0;
  else if (key == 5) x->force_bn = value;
  else if (key == 6) x->p2p_on_lane = value ? 1 : 0;
  else if (key == 7) x->force_cg = value;
  else if (key == 8) x->force_sk = value;
  else if (key == 9) x->bwd_sm_reserve = value < 0 ? 0 : (value > 120 ? 120 : value);
  else if (key == 10) x->sm_reserve = value < 0 ? 0 : (value > 120 ? 120 : value);
  else return fail(FLOWMOE_ERR_INVALID, "flowmoe_debug_set: unknown key");
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_profile_begin(flowmoe_ctx* x) {
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  x->prof.recs.clear();
  x->prof.used = 0;
  x->prof.on = true;
  return FLOWMOE_OK;
}

int flowmoe_profile_end(flowmoe_ctx* x, flowmoe_prof_entry* out, int max_entries) {
  if (!x) {
    fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
    return -1;
  }
  Prof& pr = x->prof;
  pr.on = false;
  if (cudaDeviceSynchronize() != cudaSuccess) {
    fail(FLOWMOE_ERR_CUDA, "flowmoe_profile_end: device synchronize failed");
    return -1;
  }
  std::vector<flowmoe_prof_entry> agg(KK_COUNT);
  for (int i = 0; i < KK_COUNT; ++i) agg[i] = {KK_NAMES[i], 0, 0.0, 0.0, 0.0};
  for (const ProfRec& r : pr.recs) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pr.pool[r.ev], pr.pool[r.ev + 1]);
    agg[r.kind].launches += 1;
    agg[r.kind].ms += ms;
    agg[r.kind].flops += r.flops;
    agg[r.kind].bytes += r.bytes;
  }
  int n = 0;
  for (int i = 0; i < KK_COUNT; ++i)
    if (agg[i].launches > 0 && n < max_entries && out) out[n++] = agg[i];
  pr.recs.clear();
  pr.used = 0;
  return n;
}

flowmoe_status flowmoe_tasklog_begin(flowmoe_ctx* x) {
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  FM_CUDA(cudaDeviceSynchronize());
  TaskLog& tl = x->tlog;
  std::lock_guard<std::mutex> lk(tl.mu);
  if (!tl.base) FM_CUDA(cudaEventCreate(&tl.base));
  FM_CUDA(cudaEventRecord(tl.base, x->s_comp));
  tl.recs.clear();
  tl.used = 0;
  tl.fwd_seq = tl.bwd_seq = 0;
  tl.on = true;
  return FLOWMOE_OK;
}

int flowmoe_tasklog_end(flowmoe_ctx* x, flowmoe_task_rec* out, int max_entries) {
  if (!x) {
    fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
    return -1;
  }
  TaskLog& tl = x->tlog;
  tl.on = false;
  if (cudaDeviceSynchronize() != cudaSuccess) {
    fail(FLOWMOE_ERR_CUDA, "flowmoe_tasklog_end: device synchronize failed");
    return -1;
  }
  std::lock_guard<std::mutex> lk(tl.mu);
  int n = 0;
  for (const TaskRec& r : tl.recs) {
    if (!out || n >= max_entries) break;
    float t0 = 0.f, t1 = 0.f;
    cudaEventElapsedTime(&t0, tl.base, tl.pool[r.ev]);
    cudaEventElapsedTime(&t1, tl.base, tl.pool[r.ev + 1]);
    out[n++] = {r.kind, r.block, r.chunk, r.dir, r.stream, (double)t0, (double)t1};
  }
  tl.recs.clear();
  tl.used = 0;
  return n;
}

flowmoe_status flowmoe_get_unique_id(uint8_t id[128]) {
  if (!id) return fail(FLOWMOE_ERR_INVALID, "id is NULL");
  ncclUniqueId u;
  FM_NCCL(ncclGetUniqueId(&u));
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  memcpy(id, &u, 128);
  return FLOWMOE_OK;
}

}  // extern "C"

namespace {
int ar_max_ctas() {
  const char* e = getenv("FLOWMOE_AR_MAX_CTAS");
  const int v = e ? atoi(e) : 0;
  return v > 0 ? v : 32;
}

// `g` non-null: a member of the in-process simulated world (no NCCL; peers wired later)
flowmoe_status create_impl(const flowmoe_config* cfg, const uint8_t id[128], int device, LocalGroup* g,
                           flowmoe_ctx** out) {
  if (!out) return fail(FLOWMOE_ERR_INVALID, "out is NULL");
  *out = nullptr;
  if (flowmoe_status s = validate(cfg)) return s;
  if (cfg->world_size > 1 && !id && !g) return fail(FLOWMOE_ERR_INVALID, "id is NULL with world_size > 1");
  auto* x = new flowmoe_ctx();
  x->cfg = *cfg;
  x->group = g;
  // VANILLA_EP treats the block as one chunk (R = 1); PIPE_MOE and FLOWMOE_AR keep the
  // MHA+gate task AT unsplit; only FLOWMOE_AR and FLOWMOE pipeline the AR (Table 6)
  if (cfg->schedule == FLOWMOE_SCHED_VANILLA_EP) x->cfg.R = 1;
  x->at_split = cfg->schedule == FLOWMOE_SCHED_FLOWMOE || cfg->schedule == FLOWMOE_SCHED_FLOWMOE_AT;
  x->ar_pipelined = cfg->schedule == FLOWMOE_SCHED_FLOWMOE || cfg->schedule == FLOWMOE_SCHED_FLOWMOE_AR;
  x->dev = device;
  x->T = cfg->B;
  x->Tr = cfg->B / x->cfg.R;
  x->N = cfg->seq_len;
  x->S = cfg->B / cfg->seq_len;
  x->M = cfg->M;
  x->E = cfg->E;
  x->k = cfg->top_k;
  x->H = cfg->n_heads;
  x->F = cfg->d_ffn;
  x->P = cfg->world_size;
  x->El = cfg->E / cfg->world_size;
  x->C = capacity_of(&x->cfg, x->Tr);
  x->tok = x->at_split && x->Tr < x->N;
  x->dt = cfg->dtype == FLOWMOE_BF16 ? DT_BF16 : DT_F32;
  x->es = cfg->dtype == FLOWMOE_BF16 ? 2 : 4;
  x->L = layout_of(x);
  auto cleanup_fail = [&](flowmoe_status s) {
    flowmoe_destroy(x);
    return s;
  };
  if (cudaSetDevice(device) != cudaSuccess)
    return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "cudaSetDevice failed"));
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);  // hi = greatest priority (numerically lowest)
  if (cudaStreamCreateWithPriority(&x->s_comp, cudaStreamNonBlocking, 0) ||
      cudaStreamCreateWithPriority(&x->s_a2a, cudaStreamNonBlocking, hi) ||
      cudaStreamCreateWithPriority(&x->s_ar, cudaStreamNonBlocking, lo))
    return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "stream creation failed"));
  auto mk = [&](cudaEvent_t* e) { return cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess; };
  {
    const int R_ = x->cfg.R;
    const int nl = cfg->compute_streams < 1 ? 1 : (cfg->compute_streams > R_ ? R_ : cfg->compute_streams);
    x->lanes.push_back(x->s_comp);
    for (int l = 1; l < nl; ++l) {
      cudaStream_t st = nullptr;
      if (cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, 0))
        return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "stream creation failed"));
      x->lanes.push_back(st);
    }
    if (nl > 1) {
      if (cudaStreamCreateWithPriority(&x->s_wg, cudaStreamNonBlocking, 0))
        return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "stream creation failed"));
    } else {
      x->s_wg = x->s_comp;
    }
    x->ev_lane.resize(nl);
    for (auto& e : x->ev_lane)
      if (!mk(&e)) return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "event creation failed"));
  }
  x->atb_cap.assign(x->cfg.R, 0);
  x->atb_rec.assign(x->cfg.R, 0);
  for (auto* v : {&x->ev_at, &x->ev_d, &x->ev_e, &x->ev_c, &x->ev_cb, &x->ev_cba, &x->ev_eb, &x->ev_dba,
                  &x->ev_qkv, &x->ev_dctx, &x->ev_atb}) {
    v->resize(x->cfg.R);
    for (auto& e : *v)
      if (!mk(&e)) return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "event creation failed"));
  }
  if (g) {
    x->ev_sent.resize(4 * x->cfg.R);
    for (auto& e : x->ev_sent)
      if (!mk(&e)) return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "event creation failed"));
  }
  x->ticket_ev.resize(NUM_TICKET_EVENTS);
  for (auto& e : x->ticket_ev)
    if (!mk(&e)) return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "event creation failed"));
  if (!mk(&x->ev_in) || !mk(&x->ev_done) || !mk(&x->ev_grads_a) || !mk(&x->ev_grads_b) ||
      !mk(&x->ev_bwd_done))
    return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "event creation failed"));
  // backward workspaces
  auto alloc = [&](void** p, size_t bytes) {
    if (cudaMalloc(p, bytes < 256 ? 256 : bytes) != cudaSuccess) return false;
    x->allocs.push_back(*p);
    return true;
  };
  const size_t es = x->es;
  const int64_t R = x->cfg.R, ECM = x->E * x->C * x->M;
  bool ok = alloc((void**)&x->route_done, R * sizeof(unsigned int)) &&
            cudaMemset(x->route_done, 0, R * sizeof(unsigned int)) == cudaSuccess &&
            alloc(&x->dxe, R * ECM * es) && alloc(&x->dctx, x->T * x->M * es) &&
            alloc((void**)&x->dw, x->T * x->k * 4) && alloc((void**)&x->Dbuf, x->T * x->H * 4) &&
            alloc((void**)&x->wg_part, gate_wgrad_scratch_floats((int)x->T, (int)x->M, (int)x->E) * 4);
  const int nsets = x->s_wg != x->s_comp ? 2 : 1;
  for (int st = 0; st < nsets && ok; ++st) {
    ok = alloc(&x->ws_dyc[st], R * ECM * es) && alloc(&x->ws_dz[st], (size_t)R * x->E * x->C * x->F * es) &&
         alloc(&x->ws_dA[st], x->T * x->M * es) && alloc(&x->ws_dqkv[st], x->T * 3 * x->M * es) &&
         alloc((void**)&x->ws_dl[st], x->T * x->E * 4);
    x->ws_dye[st] = x->ws_dyc[st];  // P > 1 receives dY into the per-block saved stash
    if (ok && !mk(&x->ev_wg_done[st])) return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "event creation failed"));
  }
  for (int st = nsets; st < 2; ++st) {
    x->ws_dyc[st] = x->ws_dyc[0]; x->ws_dye[st] = x->ws_dye[0]; x->ws_dz[st] = x->ws_dz[0];
    x->ws_dA[st] = x->ws_dA[0]; x->ws_dqkv[st] = x->ws_dqkv[0]; x->ws_dl[st] = x->ws_dl[0];
  }
  if (ok && x->P > 1) ok = alloc(&x->dxc, R * ECM * es);
  if (!ok) return cleanup_fail(fail(FLOWMOE_ERR_OOM, "workspace allocation failed"));
  if (x->P == 1) x->dxc = x->dxe;
  for (size_t i = 0; i < x->lanes.size() && ok && x->dt == DT_BF16; ++i) {
    float* w = nullptr;
    unsigned int* t = nullptr;
    ok = alloc((void**)&w, SK_WS_FLOATS * 4) && alloc((void**)&t, SK_TICKS * 4) &&
         cudaMemset(t, 0, SK_TICKS * 4) == cudaSuccess;
    x->sk_ws.push_back(w);
    x->sk_tick.push_back(t);
  }
  if (!ok) return cleanup_fail(fail(FLOWMOE_ERR_OOM, "workspace allocation failed"));
  if (x->dt == DT_BF16 && gemm_tc_init() != 0)
    return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "cuTensorMapEncodeTiled entry point unavailable"));
  if (x->P > 1 && !g) {
    if (!alloc(&x->xchg, (x->P + 2) * sizeof(IpcRec)))
      return cleanup_fail(fail(FLOWMOE_ERR_OOM, "workspace allocation failed"));
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclConfig_t nc = NCCL_CONFIG_INITIALIZER;
    nc.blocking = 1;
    if (ncclCommInitRankConfig(&x->comm_a2a, (int)x->P, u, cfg->rank, &nc) != ncclSuccess)
      return cleanup_fail(fail(FLOWMOE_ERR_NCCL, "ncclCommInitRankConfig failed"));
    // the AR communicator runs in the gaps of the compute: cap its CTAs so a long AR chunk
    // never takes more than a few SMs from the compute lanes
    ncclConfig_t nc2 = NCCL_CONFIG_INITIALIZER;
    nc2.blocking = 1;
    nc2.maxCTAs = ar_max_ctas();
    // and the backward GEMMs (persistent grids: one CTA per SM) leave as many SMs free, so
    // an AR chunk's CTAs start at once instead of after the GEMM holding their SMs
    // (dsv2s N=2: 9.23 -> 9.03 ms; key 9 overrides)
    x->bwd_sm_reserve = ar_max_ctas();
    if (ncclCommSplit(x->comm_a2a, 0, cfg->rank, &x->comm_ar, &nc2) != ncclSuccess)
      return cleanup_fail(fail(FLOWMOE_ERR_NCCL, "ncclCommSplit failed"));
    x->a2a_comm.push_back(x->comm_a2a);
  }
  if (x->P > 1) x->a2a_stream.push_back(x->s_a2a);
  if (x->P > 1 && (g || cfg->a2a_impl == FLOWMOE_A2A_P2P)) {
    const size_t nfl = (size_t)4 * x->cfg.R * x->P;
    const size_t bytes = (2 * nfl + 8 * x->cfg.R + 1) * sizeof(unsigned int);
    if (!alloc(&x->p2p_arena, bytes) || cudaMemset(x->p2p_arena, 0, bytes) != cudaSuccess ||
        cudaDeviceSynchronize() != cudaSuccess)
      return cleanup_fail(fail(FLOWMOE_ERR_OOM, "p2p arena allocation failed"));
    x->flags = reinterpret_cast<unsigned int*>(x->p2p_arena);
    x->piece_cnt = x->flags + nfl;
    x->seen = x->piece_cnt + nfl;
    x->p2p_err = x->seen + 4 * x->cfg.R;
    x->grid_cnt = x->p2p_err + 1;
    if (!g) {
      std::vector<void*> v;
      if (ipc_exchange(x, x->p2p_arena, &v, &x->ipc_opened) != FLOWMOE_OK)
        return cleanup_fail(FLOWMOE_ERR_CUDA);
      for (void* q : v) x->peer_flags.push_back(reinterpret_cast<unsigned int*>(q));
      if (ipc_exchange(x, x->dxc, &x->peer_dxc, &x->ipc_opened) != FLOWMOE_OK) return cleanup_fail(FLOWMOE_ERR_CUDA);
      x->p2p = true;
    }
  }
  // A2A lanes (NCCL path only: the peer-memory exchanges run on the compute lanes)
  for (size_t l = 1; l < x->lanes.size() && x->P > 1 && !x->p2p && !g; ++l) {
    ncclConfig_t nc3 = NCCL_CONFIG_INITIALIZER;
    nc3.blocking = 1;
    ncclComm_t c2 = nullptr;
    cudaStream_t s2 = nullptr;
    if (ncclCommSplit(x->comm_a2a, 0, cfg->rank, &c2, &nc3) != ncclSuccess)
      return cleanup_fail(fail(FLOWMOE_ERR_NCCL, "ncclCommSplit (A2A lane) failed"));
    x->a2a_comm.push_back(c2);
    if (cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, hi))
      return cleanup_fail(fail(FLOWMOE_ERR_CUDA, "stream creation failed"));
    x->a2a_stream.push_back(s2);
  }
  *out = x;
  return FLOWMOE_OK;
}

// collective registration of one saved stash (NCCL world: CUDA-IPC exchange with
// agreement; simulated world: record it, peers resolved once every rank registered)
flowmoe_status register_saved(flowmoe_ctx* x, const void* saved) {
  if (x->P == 1 || !x->p2p || x->peer_saved.count(saved)) return FLOWMOE_OK;
  if (LocalGroup* g = x->group) {
    std::lock_guard<std::mutex> lk(g->mu);
    auto& mine = g->saved[x->cfg.rank];
    size_t n = 0;
    while (n < mine.size() && mine[n] != saved) ++n;
    if (n == mine.size()) mine.push_back(saved);
    for (int q = 0; q < g->P; ++q)
      if (g->saved[q].size() <= n) return FLOWMOE_OK;  // resolved when the last rank registers
    for (int q = 0; q < g->P; ++q) {  // every rank's n-th stash is now known
      std::vector<void*> v(g->P);
      for (int q2 = 0; q2 < g->P; ++q2) v[q2] = const_cast<void*>(g->saved[q2][n]);
      g->m[q]->peer_saved[g->saved[q][n]] = v;
    }
    return FLOWMOE_OK;
  }
  std::vector<void*> v, opened;
  if (flowmoe_status st = ipc_exchange(x, const_cast<void*>(saved), &v, &opened)) return st;
  x->peer_saved[saved] = v;
  x->saved_opened[saved] = opened;
  x->saved_order.push_back(saved);
  return FLOWMOE_OK;
}
}  // namespace

extern "C" {

flowmoe_status flowmoe_create(const flowmoe_config* cfg, const uint8_t id[128], int device,
                              flowmoe_ctx** out) {
  return create_impl(cfg, id, device, nullptr, out);
}

flowmoe_status flowmoe_register_saved(flowmoe_ctx* x, const void* saved) {
  if (!x || !saved) return fail(FLOWMOE_ERR_INVALID, "register_saved: NULL argument");
  return register_saved(x, saved);
}

flowmoe_status flowmoe_unregister_saved(flowmoe_ctx* x, const void* saved) {
  if (!x || !saved) return fail(FLOWMOE_ERR_INVALID, "unregister_saved: NULL argument");
  if (x->group) return fail(FLOWMOE_ERR_UNSUPPORTED, "unregister_saved: not supported in a local group");
  auto it = x->saved_opened.find(saved);
  if (it != x->saved_opened.end()) {
    FM_CUDA(cudaDeviceSynchronize());  // no enqueued exchange may still target the mapping
    for (void* pb : it->second) cudaIpcCloseMemHandle(pb);
    x->saved_opened.erase(it);
  }
  x->peer_saved.erase(saved);
  for (size_t i = 0; i < x->saved_order.size(); ++i)
    if (x->saved_order[i] == saved) { x->saved_order.erase(x->saved_order.begin() + i); break; }
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_test_exchange(flowmoe_ctx* x, void* saved, int kind, int r, int iters, cudaStream_t stream) {
  if (!x || !saved) return fail(FLOWMOE_ERR_INVALID, "test_exchange: NULL argument");
  if (kind < 0 || kind > 1 || r < 0 || r >= x->cfg.R || iters < 1)
    return fail(FLOWMOE_ERR_INVALID, "test_exchange: kind in {0,1}, 0 <= r < R, iters >= 1");
  if (x->P == 1 || x->group) return fail(FLOWMOE_ERR_UNSUPPORTED, "test_exchange: needs world_size > 1 (NCCL world)");
  apply_ctx(x);
  bool use_p2p = false;
  if (flowmoe_status st = resolve_p2p(x, saved, stream, &use_p2p)) return st;
  const SavedLayout& L = x->L;
  const size_t src = kind == 0 ? L.send : L.ye, dst = kind == 0 ? L.xe : L.yc;
  cudaStream_t sa = use_p2p ? stream : x->a2a_stream[r % x->a2a_stream.size()];
  if (sa != stream) {
    FM_CUDA(cudaEventRecord(x->ev_in, stream));
    FM_CUDA(cudaStreamWaitEvent(sa, x->ev_in, 0));
  }
  for (int i = 0; i < iters; ++i) {
    if (use_p2p) {
      std::vector<void*> d(x->P);
      for (int q = 0; q < x->P; ++q) d[q] = (char*)x->peer_saved[saved][q] + dst;
      if (flowmoe_status st = p2p_exchange(x, kind, r, (char*)saved + src, d.data(), kind == 0 ? 1 : 0, sa)) return st;
    } else if (kind == 0) {
      if (flowmoe_status st = a2a_to_experts(x, (char*)saved + src, (char*)saved + dst, r)) return st;
    } else if (flowmoe_status st = a2a_to_owners(x, (char*)saved + src, (char*)saved + dst, r)) {
      return st;
    }
  }
  if (sa != stream) {
    FM_CUDA(cudaEventRecord(x->ev_done, sa));
    FM_CUDA(cudaStreamWaitEvent(stream, x->ev_done, 0));
  }
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_test_arrivals(const flowmoe_ctx* x, unsigned int* out, size_t n) {
  if (!x || !out) return fail(FLOWMOE_ERR_INVALID, "test_arrivals: NULL argument");
  const size_t nfl = (size_t)4 * x->cfg.R * x->P;
  if (!x->flags) return fail(FLOWMOE_ERR_STATE, "test_arrivals: no peer-memory A2A in this ctx");
  if (n < nfl) return fail(FLOWMOE_ERR_INVALID, "test_arrivals: need 4*R*world_size entries");
  FM_CUDA(cudaDeviceSynchronize());
  FM_CUDA(cudaMemcpy(out, x->flags, nfl * sizeof(unsigned int), cudaMemcpyDeviceToHost));
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_check_health(flowmoe_ctx* x) {
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (x->p2p_err) {
    unsigned int e = 0;
    if (cudaMemcpy(&e, x->p2p_err, sizeof(e), cudaMemcpyDeviceToHost) != cudaSuccess)
      return fail(FLOWMOE_ERR_CUDA, std::string("device fault (a peer-memory A2A wait that timed out traps): ") +
                                        cudaGetErrorString(cudaGetLastError()));
    if (e) return fail(FLOWMOE_ERR_STATE, "peer-memory A2A timed out waiting for a peer");
  }
  ncclResult_t a = ncclSuccess;
  for (ncclComm_t c : x->a2a_comm) {
    ncclResult_t e = ncclSuccess;
    if (c) ncclCommGetAsyncError(c, &e);
    if (e != ncclSuccess) a = e;
  }
  if (x->comm_ar) {
    ncclResult_t e = ncclSuccess;
    ncclCommGetAsyncError(x->comm_ar, &e);
    if (e != ncclSuccess) a = e;
  }
  if (a != ncclSuccess) return fail(FLOWMOE_ERR_NCCL, std::string("async NCCL error: ") + ncclGetErrorString(a));
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_create_local_group(const flowmoe_config* cfg, int P, int device, flowmoe_ctx** out) {
  if (!cfg || !out) return fail(FLOWMOE_ERR_INVALID, "create_local_group: NULL argument");
  if (P < 2 || P > 8) return fail(FLOWMOE_ERR_INVALID, "create_local_group: P must be in [2, 8]");
  if (cfg->schedule != FLOWMOE_SCHED_FLOWMOE && cfg->schedule != FLOWMOE_SCHED_FLOWMOE_AR)
    return fail(FLOWMOE_ERR_UNSUPPORTED, "create_local_group: only the per-block (pipelined) AR schedules");
  for (int q = 0; q < P; ++q) out[q] = nullptr;
  auto* g = new LocalGroup();
  g->P = P;
  g->m.assign(P, nullptr);
  g->saved.resize(P);
  g->subs.resize(P);
  g->ticket_sub.resize(P);
  g->ticket_done.resize(P);
  for (int q = 0; q < P; ++q) {
    flowmoe_config c = *cfg;
    c.world_size = P;
    c.rank = q;
    c.a2a_impl = FLOWMOE_A2A_P2P;
    flowmoe_status st = create_impl(&c, nullptr, device, g, &out[q]);
    if (st) {
      const std::string msg = g_err;
      for (int q2 = 0; q2 < q; ++q2) flowmoe_destroy(out[q2]);
      return fail(st, msg);
    }
    g->m[q] = out[q];
  }
  for (int q = 0; q < P; ++q) {
    flowmoe_ctx* x = out[q];
    for (int q2 = 0; q2 < P; ++q2) {
      x->peer_flags.push_back(out[q2]->flags);
      x->peer_dxc.push_back(out[q2]->dxc);
    }
    x->p2p = true;
  }
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  FM_CUDA(cudaStreamCreateWithPriority(&g->s, cudaStreamNonBlocking, lo));
  return FLOWMOE_OK;
}

size_t flowmoe_saved_bytes(const flowmoe_ctx* x) { return x ? x->L.total : 0; }

size_t flowmoe_grad_flat_count(const flowmoe_ctx* x) {
  return x ? (size_t)(4 * x->M * x->M + x->M * x->E) : 0;
}

flowmoe_status flowmoe_saved_routing_offsets(const flowmoe_ctx* x, size_t* logits, size_t* idx,
                                             size_t* w, size_t* pos, size_t* counts) {
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (logits) *logits = x->L.logits;
  if (idx) *idx = x->L.idx;
  if (w) *w = x->L.w;
  if (pos) *pos = x->L.pos;
  if (counts) *counts = x->L.counts;
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_set_forced_routing(flowmoe_ctx* x, const int32_t* idx) {
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  x->forced = idx;
  return FLOWMOE_OK;
}

}  // extern "C"

namespace {
// Simulated world: host-side rendezvous of the P member threads (each rank is driven by its
// own host thread, e.g. a Python thread: ctypes releases the GIL).  false on timeout.
bool group_barrier(LocalGroup* g) {
  std::unique_lock<std::mutex> lk(g->mu);
  const uint64_t gen = g->bar_gen;
  if (++g->bar_count == g->P) {
    g->bar_count = 0;
    ++g->bar_gen;
    g->cv.notify_all();
    return true;
  }
  return g->cv.wait_for(lk, std::chrono::seconds(120), [&] { return g->bar_gen != gen; });
}

// One peer-memory exchange (kind 0 D_r, 1 C_r, 2 C_r^bwd, 3 D_r^bwd) of chunk r on stream sa:
// this rank's CTAs store its C×M blocks into every destination's receive buffer and bump
// the destinations' arrival counters.  Across GPUs the completing CTA then waits (acquire)
// for every source's arrival.  In the simulated world no kernel ever waits for another
// launch (nothing guarantees that separate launches on one GPU run at the same time): the
// send kernel records an event, the member threads meet at a host barrier, and the stream
// waits for every peer's send event instead; a second barrier keeps any member from
// re-recording its event before every peer has enqueued its wait.
flowmoe_status p2p_exchange(flowmoe_ctx* x, int kind, int r, const void* src, void* const* dst, int to_experts,
                            cudaStream_t sa) {
  const int R = x->cfg.R;
  const int64_t blk = x->C * x->M * (int64_t)x->es;
  LocalGroup* g = x->group;
  FM_K(1, a2a_p2p(src, dst, x->peer_flags.data(), x->piece_cnt, x->flags, x->seen, x->p2p_err, kind, r, R,
                  (int)x->P, (int)x->El, x->cfg.rank, to_experts, blk, sa, sa, true, g == nullptr,
                  g ? nullptr : x->grid_cnt));
  if (!g) return FLOWMOE_OK;
  cudaEvent_t ev = x->ev_sent[kind * R + r];
  FM_CUDA(cudaEventRecord(ev, sa));
  if (!group_barrier(g)) return fail(FLOWMOE_ERR_STATE, "local group: a peer did not reach the exchange (120 s)");
  for (int q = 0; q < g->P; ++q)
    if (q != x->cfg.rank) FM_CUDA(cudaStreamWaitEvent(sa, g->m[q]->ev_sent[kind * R + r], 0));
  if (!group_barrier(g)) return fail(FLOWMOE_ERR_STATE, "local group: a peer did not reach the exchange (120 s)");
  return FLOWMOE_OK;
}
}  // namespace

namespace {
// One block's forward.  fork: lanes first wait for `stream`; join: `stream` then waits for
// every lane.  The stack API forks once and joins once, so chunk r of block l+1 follows
// chunk r of block l on lane r % n without a block-boundary barrier.
flowmoe_status enqueue_fwd(flowmoe_ctx* x, const flowmoe_params* p, const void* xin, void* y, void* saved,
                           cudaStream_t stream, bool fork, bool join) {
  if (!x || !p || !xin || !y || !saved) return fail(FLOWMOE_ERR_INVALID, "block_fwd: NULL argument");
  if (!p->wqkv || !p->wo || !p->wg || !p->w1 || !p->b1 || !p->w2 || !p->b2)
    return fail(FLOWMOE_ERR_INVALID, "block_fwd: NULL parameter pointer");
  x->gemm_max_sms = x->sm_reserve > 0 ? 148 - x->sm_reserve : 0;
  const int dt = x->dt;
  const size_t es = x->es;
  const int R = x->cfg.R;
  const int64_t M = x->M, E = x->E, k = x->k, C = x->C, F = x->F, Tr = x->Tr, El = x->El, P = x->P;
  const int64_t ECM = E * C * M, PC = P * C, ldE = R * C;
  const SavedLayout& L = x->L;
  // the per-kernel profile (flowmoe_profile_begin) collapses the lanes so that each
  // kernel's event-timed duration is its own, not shared with co-running chunks
  const int nl = x->prof.on ? 1 : (int)x->lanes.size();
  bool use_p2p = false;
  if (flowmoe_status st = resolve_p2p(x, saved, stream, &use_p2p)) return st;
  if (fork)
    if (flowmoe_status st = fork_lanes(x, stream)) return st;
  // Unsplit AT (PIPE_MOE, FLOWMOE_AR) reads all T rows of x on lane 0; inside a stack
  // (no fork) the previous block wrote chunk r of x on lane r, so join the lanes first.
  if (!fork && !x->at_split && nl > 1)
    if (flowmoe_status st = join_lanes(x, x->lanes[0])) return st;
  if (x->tlog.on) { x->tlog.block = x->tlog.fwd_seq++; x->tlog.dir = 0; }
  // ---- AT_1..AT_R (Eq.(3)): MHA + gate + route + pack into the dispatch send buffer.
  // Policies that keep AT unsplit (PIPE_MOE, FLOWMOE_AR) run MHA + gate once over all
  // tokens, then route/pack per chunk (capacity is per chunk in every policy).
  const int n_at = x->at_split ? R : 1;
  const int64_t Ta = x->at_split ? Tr : x->T;
  for (int ai = 0; ai < n_at; ++ai) {
    cudaStream_t sc = x->lanes[ai % nl];
    const int64_t t0 = ai * Ta;
    const char* xr = (const char*)xin + t0 * M * es;
    void* qkv = at<char>(saved, L.qkv + t0 * 3 * M * es);
    void* ctxb = at<char>(saved, L.ctx + t0 * M * es);
    void* a = at<char>(saved, L.a + t0 * M * es);
    const int tk_at = task_begin(x, sc);
    GemmArgs g;
    g.M = (int)Ta; g.N = (int)(3 * M); g.K = (int)M;
    g.A = xr; g.lda = M; g.B = p->wqkv; g.ldb = 3 * M; g.C = qkv; g.ldc = 3 * M;
    FM_GEMM(KK_QKV, g);
    // attention rows: whole sequences of the chunk, or (token chunk) positions
    // [p0, p0+Ta) of sequence t0/N attending to that sequence's keys before them
    int64_t a0 = t0, nseq = Ta / x->N, p0 = 0, np = x->N;
    double attn_flops = 4.0 * Ta * x->N * M * (x->cfg.causal ? 0.5 : 1.0);
    if (x->tok) {
      a0 = t0 / x->N * x->N; nseq = 1; p0 = t0 - a0; np = Ta;
      attn_flops = 4.0 * M * ((double)Ta * p0 + 0.5 * Ta * Ta);
      FM_CUDA(cudaEventRecord(x->ev_qkv[ai], sc));
      for (int64_t q = a0 / Ta; q < ai; ++q)  // earlier chunks of the sequence
        if (x->lanes[q % nl] != sc) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_qkv[q], 0));
    }
    FM_KP(KK_ATTN_F, 1, attn_flops, (double)Ta * 5 * M * es + Ta * x->H * 4.0, sc,
          attn_fwd(dt, at<char>(saved, L.qkv + a0 * 3 * M * es), at<char>(saved, L.ctx + a0 * M * es),
                   at<float>(saved, L.lse + a0 * x->H * 4), (int)nseq, (int)x->N, (int)p0, (int)np, (int)M,
                   (int)x->H, x->cfg.causal, sc));
    g = GemmArgs();
    g.M = (int)Ta; g.N = (int)M; g.K = (int)M;
    g.A = ctxb; g.lda = M; g.B = p->wo; g.ldb = M; g.C = a; g.ldc = M;
    if (x->cfg.residual) { g.resid = xr; g.ldr = M; }
    FM_GEMM(KK_OPROJ, g);
    if (x->at_split) {  // gate + routing scan of chunk ai in one launch (last-CTA scan)
      FM_KP(KK_GATE, 1, 2.0 * Ta * M * E, (double)Ta * M * es + M * E * es + Ta * E * 4.0 + Ta * k * 20.0, sc,
            gate_route(dt, a, p->wg, x->forced ? x->forced + t0 * k : nullptr, at<float>(saved, L.logits + t0 * E * 4),
                       at<int32_t>(saved, L.idx + t0 * k * 4), at<float>(saved, L.w + t0 * k * 4),
                       at<int32_t>(saved, L.pos + t0 * k * 4), at<int32_t>(saved, L.counts + ai * E * 4),
                       at<int32_t>(saved, L.src + ai * E * C * 4), x->route_done + ai, (int)Ta, (int)M, (int)E,
                       (int)k, (int)C, sc));
    } else {
      FM_KP(KK_GATE, 1, 2.0 * Ta * M * E, (double)Ta * M * es + M * E * es + Ta * E * 4.0 + Ta * k * 8.0, sc,
            gate_topk(dt, a, p->wg, x->forced ? x->forced + t0 * k : nullptr, at<float>(saved, L.logits + t0 * E * 4),
                      at<int32_t>(saved, L.idx + t0 * k * 4), at<float>(saved, L.w + t0 * k * 4), (int)Ta, (int)M,
                      (int)E, (int)k, sc));
    }
   for (int r = x->at_split ? ai : 0; r < (x->at_split ? ai + 1 : R); ++r) {
    const int64_t t0 = r * Tr;
    void* a = at<char>(saved, L.a + t0 * M * es);
    int32_t* src = at<int32_t>(saved, L.src + r * E * C * 4);
    if (!x->at_split)
      FM_KP(KK_ROUTE, 1, 0, Tr * k * 12.0 + E * C * 4.0 + E * 4.0, sc,
            route_scan(at<int32_t>(saved, L.idx + t0 * k * 4), at<int32_t>(saved, L.pos + t0 * k * 4),
                       at<int32_t>(saved, L.counts + r * E * 4), src, (int)Tr, (int)E, (int)k, (int)C, sc));
    FM_KP(KK_PACK, 1, 0, 2.0 * E * C * M * es, sc,
          permute_pack(dt, a, src, at<char>(saved, L.send + r * C * M * es), (int)E, (int)C, (int)ldE, (int)M,
                       (int)k, sc));
    // the task's end marker before the event D_r waits on: a marker recorded after the
    // release can be stamped later than the waiting stream's start (front-end skew)
    if (x->at_split) task_end(x, tk_at, TK_AT, ai, sc);
    FM_CUDA(cudaEventRecord(x->ev_at[r], sc));
   }
    if (!x->at_split) task_end(x, tk_at, TK_AT, -1, sc);
  }
  // ---- D_1..D_R (Eq.(4)) on the high-priority A2A stream
  if (P > 1)
    for (int r = 0; r < R; ++r) {
      cudaStream_t sa = (use_p2p && g_p2p_on_lane) ? x->lanes[r % nl] : x->a2a_stream[r % x->a2a_stream.size()];
      FM_CUDA(cudaStreamWaitEvent(sa, x->ev_at[r], 0));
      const int tk = task_begin(x, sa);
      int pi = prof_start(sa);
      if (use_p2p) {
        std::vector<void*> dst(P);
        for (int q = 0; q < P; ++q) dst[q] = (char*)x->peer_saved[saved][q] + L.xe;
        if (flowmoe_status st_ = p2p_exchange(x, 0, r, at<char>(saved, L.send), dst.data(), 1, sa)) return st_;
      } else if (flowmoe_status s = a2a_to_experts(x, at<char>(saved, L.send), at<char>(saved, L.xe), r)) return s;
      prof_stop(pi, KK_A2A_D, 0, (double)ECM * es * (P - 1) / P, sa);
      task_end(x, tk, TK_D, r, sa);
      FM_CUDA(cudaEventRecord(x->ev_d[r], sa));
    }
  // ---- E_1..E_R: batched expert FFN over the [P*C] capacity rows of chunk r of each local expert
  for (int r = 0; r < R; ++r) {
    cudaStream_t sc = x->lanes[r % nl];
    if (P > 1) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_d[r], 0));
    else if (!x->at_split && sc != x->lanes[0]) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_at[r], 0));
    const int tk_e = task_begin(x, sc);
    GemmArgs g;
    g.batch = (int)El; g.M = (int)PC; g.N = (int)F; g.K = (int)M;
    g.A = at<char>(saved, L.xe + r * PC * M * es); g.lda = M; g.sA = R * PC * M;
    g.B = p->w1; g.ldb = F; g.sB = M * F;
    g.C = at<char>(saved, L.h + r * PC * F * es); g.ldc = F; g.sC = R * PC * F;
    g.bias = p->b1; g.sBias = F;
    g.aux = at<char>(saved, L.z + r * PC * F * es); g.ldaux = F; g.sAux = R * PC * F;
    g.epi = EPI_BIAS_GELU_G;  // saves GELU'(Z) for the backward (L.z)
    FM_GEMM(KK_E1, g);
    g = GemmArgs();
    g.batch = (int)El; g.M = (int)PC; g.N = (int)M; g.K = (int)F;
    g.A = at<char>(saved, L.h + r * PC * F * es); g.lda = F; g.sA = R * PC * F;
    g.B = p->w2; g.ldb = M; g.sB = F * M;
    g.C = at<char>(saved, L.ye + r * PC * M * es); g.ldc = M; g.sC = R * PC * M;
    g.bias = p->b2; g.sBias = M;
    FM_GEMM(KK_E2, g);
    task_end(x, tk_e, TK_E, r, sc);
    if (P > 1) FM_CUDA(cudaEventRecord(x->ev_e[r], sc));
  }
  // ---- C_1..C_R (Eq.(4))
  if (P > 1)
    for (int r = 0; r < R; ++r) {
      cudaStream_t sa = (use_p2p && g_p2p_on_lane) ? x->lanes[r % nl] : x->a2a_stream[r % x->a2a_stream.size()];
      FM_CUDA(cudaStreamWaitEvent(sa, x->ev_e[r], 0));
      const int tk = task_begin(x, sa);
      int pi = prof_start(sa);
      if (use_p2p) {
        std::vector<void*> dst(P);
        for (int q = 0; q < P; ++q) dst[q] = (char*)x->peer_saved[saved][q] + L.yc;
        if (flowmoe_status st_ = p2p_exchange(x, 1, r, at<char>(saved, L.ye), dst.data(), 0, sa)) return st_;
      } else if (flowmoe_status s = a2a_to_owners(x, at<char>(saved, L.ye), at<char>(saved, L.yc), r)) return s;
      prof_stop(pi, KK_A2A_C, 0, (double)ECM * es * (P - 1) / P, sa);
      task_end(x, tk, TK_C, r, sa);
      FM_CUDA(cudaEventRecord(x->ev_c[r], sa));
    }
  // ---- merge: y = Σ_j w_j Y[e_j][pos_j] (+ I')
  for (int r = 0; r < R; ++r) {
    cudaStream_t sc = x->lanes[r % nl];
    if (P > 1) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_c[r], 0));
    const int64_t t0 = r * Tr;
    const int tk = task_begin(x, sc);
    FM_KP(KK_COMBINE, 1, 2.0 * Tr * k * M, (double)Tr * k * M * es + Tr * M * es * (x->cfg.residual ? 2.0 : 1.0), sc,
          unpermute_combine(dt, at<char>(saved, L.yc + r * C * M * es), at<int32_t>(saved, L.idx + t0 * k * 4),
                            at<int32_t>(saved, L.pos + t0 * k * 4), at<float>(saved, L.w + t0 * k * 4),
                            x->cfg.residual ? at<char>(saved, L.a + t0 * M * es) : nullptr,
                            (char*)y + t0 * M * es, (int)Tr, (int)M, (int)k, (int)ldE, sc));
    task_end(x, tk, TK_MERGE, r, sc);
  }
  if (join) {
    if (flowmoe_status st = join_lanes(x, x->lanes[0])) return st;
    FM_CUDA(cudaEventRecord(x->ev_done, x->lanes[0]));
    FM_CUDA(cudaStreamWaitEvent(stream, x->ev_done, 0));
  }
  return FLOWMOE_OK;
}

flowmoe_status enqueue_bwd(flowmoe_ctx* x, const flowmoe_params* p, const void* xin, const void* saved,
                           const void* dy, void* dx, const flowmoe_grads* gr, size_t chunk_bytes,
                           flowmoe_ticket* ar, cudaStream_t stream, bool fork, bool join) {
  if (!x || !p || !xin || !saved || !dy || !gr)
    return fail(FLOWMOE_ERR_INVALID, "block_bwd: NULL argument");
  if (!gr->grad_flat || !gr->dw1 || !gr->db1 || !gr->dw2 || !gr->db2)
    return fail(FLOWMOE_ERR_INVALID, "block_bwd: NULL gradient pointer");
  if (chunk_bytes == 0 || chunk_bytes % 16)
    return fail(FLOWMOE_ERR_INVALID, "block_bwd: chunk_bytes (S_p) must be a positive multiple of 16");
  {
    const int res = (x->P > 1 && x->bwd_sm_reserve > x->sm_reserve) ? x->bwd_sm_reserve : x->sm_reserve;
    x->gemm_max_sms = res > 0 ? 148 - res : 0;
  }
  const int dt = x->dt;
  const size_t es = x->es;
  const int R = x->cfg.R;
  const int64_t M = x->M, E = x->E, k = x->k, C = x->C, F = x->F, Tr = x->Tr, El = x->El, P = x->P;
  const int64_t ECM = E * C * M, PC = P * C, ldE = R * C;
  const SavedLayout& L = x->L;
  // the per-kernel profile (flowmoe_profile_begin) collapses the lanes so that each
  // kernel's event-timed duration is its own, not shared with co-running chunks
  const int nl = x->prof.on ? 1 : (int)x->lanes.size();
  // grad_mode: every weight grad of a block is produced by exactly one kernel (the
  // expert wgrads over all chunks, the deferred K=T MHA/gate wgrads), so "overwrite"
  // is a plain store and "accumulate" a TMA reduce-add / read-modify-write.
  const int gacc = x->cfg.grad_mode == FLOWMOE_GRAD_ACCUMULATE;
  const int gepi = gacc ? EPI_ACC_F32 : EPI_STORE_F32;
  if (fork)
    if (flowmoe_status st = fork_lanes(x, stream)) return st;
  // Unsplit AT^bwd (PIPE_MOE, FLOWMOE_AR) wrote all T rows of the previous block's dx and
  // read x->dw on lane 0; inside a stack (no fork) chunk r's combine_bwd_pack on lane r
  // reads those dx rows and rewrites dw, so every lane first waits for lane 0.
  if (!fork && !x->at_split && nl > 1)
    if (flowmoe_status st = lanes_follow(x, x->lanes[0])) return st;
  const int wset = x->ev_wg_done[1] ? (int)(x->bwd_calls++ & 1) : 0;
  x->dyc = x->ws_dyc[wset]; x->dye = x->ws_dye[wset]; x->dz = x->ws_dz[wset];
  if (P > 1) x->dye = const_cast<char*>(at<char>(saved, L.dye));  // per-block landing buffer
  bool use_p2p = false;
  if (flowmoe_status st = resolve_p2p(x, saved, stream, &use_p2p)) return st;
  x->dA = x->ws_dA[wset]; x->dqkv = x->ws_dqkv[wset]; x->dl = x->ws_dl[wset];
  // the wgrads that last read this workspace set must be done; an event recorded in
  // another capture (or outside the current one) is already ordered by the graph /
  // stream boundary, and waiting on it would break the capture
  if (x->ev_wg_done[1] && x->wg_recorded[wset] && x->wg_cap_id[wset] == capture_id(stream))
    for (cudaStream_t l : x->lanes) FM_CUDA(cudaStreamWaitEvent(l, x->ev_wg_done[wset], 0));
  if (x->tlog.on) { x->tlog.block = x->tlog.bwd_seq++; x->tlog.dir = 1; }
  // ---- C_R^bwd .. C_1^bwd: pack dY = w·dO into the owner-side buffer, dw = <dO, Y>
  for (int r = R - 1; r >= 0; --r) {
    cudaStream_t sc = x->lanes[r % nl];
    const int64_t t0 = r * Tr;
    const int tk = task_begin(x, sc);
    FM_KP(KK_CBPACK, 1, 4.0 * Tr * k * M, (double)Tr * M * es + 2.0 * Tr * k * M * es, sc,
          combine_bwd_pack(dt, (const char*)dy + t0 * M * es, at<char>(saved, L.yc + r * C * M * es),
                           at<int32_t>(saved, L.idx + t0 * k * 4), at<int32_t>(saved, L.pos + t0 * k * 4),
                           at<float>(saved, L.w + t0 * k * 4), at<int32_t>(saved, L.src + r * E * C * 4),
                           (char*)x->dyc + r * C * M * es, x->dw + t0 * k, (int)Tr, (int)M, (int)k, (int)E,
                           (int)C, (int)ldE, sc));
    task_end(x, tk, TK_CBPACK, r, sc);
    if (P > 1) FM_CUDA(cudaEventRecord(x->ev_cb[r], sc));
  }
  if (P > 1)
    for (int r = R - 1; r >= 0; --r) {
      cudaStream_t sa = (use_p2p && g_p2p_on_lane) ? x->lanes[r % nl] : x->a2a_stream[r % x->a2a_stream.size()];
      FM_CUDA(cudaStreamWaitEvent(sa, x->ev_cb[r], 0));
      const int tk = task_begin(x, sa);
      int pi = prof_start(sa);
      if (use_p2p) {
        std::vector<void*> dst(P);
        for (int q = 0; q < P; ++q) dst[q] = (char*)x->peer_saved[saved][q] + L.dye;
        if (flowmoe_status st_ = p2p_exchange(x, 2, r, x->dyc, dst.data(), 1, sa)) return st_;
      } else if (flowmoe_status s = a2a_to_experts(x, x->dyc, x->dye, r)) return s;
      prof_stop(pi, KK_A2A_CB, 0, (double)ECM * es * (P - 1) / P, sa);
      task_end(x, tk, TK_CB, r, sa);
      FM_CUDA(cudaEventRecord(x->ev_cba[r], sa));
    }
  // ---- E_R^bwd .. E_1^bwd (Eq.(5)): dgrads per chunk, so D_r^bwd can start early
  for (int r = R - 1; r >= 0; --r) {
    cudaStream_t sc = x->lanes[r % nl];
    if (P > 1) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_cba[r], 0));
    const int tk_eb = task_begin(x, sc);
    // dZ = (dY·W2ᵀ) ⊙ GELU'(Z)
    GemmArgs g;
    g.batch = (int)El; g.M = (int)PC; g.N = (int)F; g.K = (int)M;
    g.A = (char*)x->dye + r * PC * M * es; g.lda = M; g.sA = R * PC * M;
    g.B = p->w2; g.ldb = M; g.sB = F * M; g.b_kmajor = 1;
    g.C = (char*)x->dz + r * PC * F * es; g.ldc = F; g.sC = R * PC * F;
    g.aux = const_cast<char*>(at<char>(saved, L.z + r * PC * F * es)); g.ldaux = F; g.sAux = R * PC * F;
    g.epi = EPI_MUL_AUX;  // dZ = dH ⊙ GELU'(Z), GELU'(Z) saved by the forward
    FM_GEMM(KK_DGELU, g);
    // dX_e = dZ·W1ᵀ  -> dispatch-bwd send buffer (expert side)
    g = GemmArgs();
    g.batch = (int)El; g.M = (int)PC; g.N = (int)M; g.K = (int)F;
    g.A = (char*)x->dz + r * PC * F * es; g.lda = F; g.sA = R * PC * F;
    g.B = p->w1; g.ldb = F; g.sB = M * F; g.b_kmajor = 1;
    g.C = (char*)x->dxe + r * PC * M * es; g.ldc = M; g.sC = R * PC * M;
    FM_GEMM(KK_DXE, g);
    task_end(x, tk_eb, TK_EB, r, sc);
    FM_CUDA(cudaEventRecord(x->ev_eb[r], sc));
  }
  if (P > 1)
    for (int r = R - 1; r >= 0; --r) {
      cudaStream_t sa = (use_p2p && g_p2p_on_lane) ? x->lanes[r % nl] : x->a2a_stream[r % x->a2a_stream.size()];
      FM_CUDA(cudaStreamWaitEvent(sa, x->ev_eb[r], 0));
      const int tk = task_begin(x, sa);
      int pi = prof_start(sa);
      if (use_p2p) {
        if (flowmoe_status st_ = p2p_exchange(x, 3, r, x->dxe, x->peer_dxc.data(), 0, sa)) return st_;
      } else if (flowmoe_status s = a2a_to_owners(x, x->dxe, x->dxc, r)) return s;
      prof_stop(pi, KK_A2A_DB, 0, (double)ECM * es * (P - 1) / P, sa);
      task_end(x, tk, TK_DB, r, sa);
      FM_CUDA(cudaEventRecord(x->ev_dba[r], sa));
    }
  // ---- expert wgrads over all R chunks at once (K = R·P·C rows), overlapping the
  // last D^bwd A2As; the sums are the chunk sums of P:1173 in a different order.
  {
    cudaStream_t sc = nl > 1 ? x->s_wg : x->lanes[0];
    for (int r = 0; r < R; ++r)
      if (sc != x->lanes[r % nl]) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_eb[r], 0));
    const int tk_wge = task_begin(x, sc);
    GemmArgs g;  // dW2 += Hᵀ·dY
    g.batch = (int)El; g.M = (int)F; g.N = (int)M; g.K = (int)(R * PC);
    g.A = at<char>(saved, L.h); g.lda = F; g.sA = R * PC * F; g.a_mmajor = 1;
    g.B = x->dye; g.ldb = M; g.sB = R * PC * M;
    g.C = gr->dw2; g.ldc = M; g.sC = F * M;
    g.epi = gepi;
    FM_GEMM(KK_DW2, g);
    FM_KP(KK_DB2, 1, (double)El * R * PC * M, (double)El * R * PC * M * es + El * M * 8.0, sc,
          colsum_acc(dt, x->dye, gr->db2, (int)El, (int)(R * PC), (int)M, gacc, sc));
    g = GemmArgs();  // dW1 += Xᵀ·dZ
    g.batch = (int)El; g.M = (int)M; g.N = (int)F; g.K = (int)(R * PC);
    g.A = at<char>(saved, L.xe); g.lda = M; g.sA = R * PC * M; g.a_mmajor = 1;
    g.B = x->dz; g.ldb = F; g.sB = R * PC * F;
    g.C = gr->dw1; g.ldc = F; g.sC = M * F;
    g.epi = gepi;
    FM_GEMM(KK_DW1, g);
    FM_KP(KK_DB1, 1, (double)El * R * PC * F, (double)El * R * PC * F * es + El * F * 8.0, sc,
          colsum_acc(dt, x->dz, gr->db1, (int)El, (int)(R * PC), (int)F, gacc, sc));
    task_end(x, tk_wge, TK_WGE, -1, sc);
  }
  // ---- AT_R^bwd .. AT_1^bwd (unsplit policies: gathers per chunk, then MHA backward
  // once over all tokens)
  const int n_atb = x->at_split ? R : 1;
  const int64_t Tb = x->at_split ? Tr : x->T;
  for (int ai = n_atb - 1; ai >= 0; --ai) {
    cudaStream_t sc = x->lanes[ai % nl];
    int tk_atb = -1;
   for (int r = x->at_split ? ai : R - 1; r >= (x->at_split ? ai : 0); --r) {
    if (P > 1) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_dba[r], 0));
    else if (sc != x->lanes[r % nl] || !x->at_split) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_eb[r], 0));
    const int64_t t0 = r * Tr;
    void* dA = (char*)x->dA + t0 * M * es;
    if (tk_atb < 0) tk_atb = task_begin(x, sc);
    FM_KP(KK_GATHER, 1, 2.0 * Tr * E * M, (double)Tr * k * M * es + Tr * M * es * (x->cfg.residual ? 2.0 : 1.0) + M * E * es, sc,
          gather_gate_bwd(dt, (char*)x->dxc + r * C * M * es, at<int32_t>(saved, L.idx + t0 * k * 4),
                          at<int32_t>(saved, L.pos + t0 * k * 4), at<float>(saved, L.w + t0 * k * 4),
                          x->dw + t0 * k, at<float>(saved, L.logits + t0 * E * 4), p->wg,
                          x->cfg.residual ? (const char*)dy + t0 * M * es : nullptr, dA, x->dl + t0 * E,
                          (int)Tr, (int)M, (int)E, (int)k, (int)ldE, sc));
   }
    const int64_t t0 = ai * Tb;
    void* dA = (char*)x->dA + t0 * M * es;
    void* dctx = (char*)x->dctx + t0 * M * es;
    void* dqkv = (char*)x->dqkv + t0 * 3 * M * es;
    int64_t a0 = t0, nseq = Tb / x->N, p0 = 0, np = x->N;
    double attn_flops = 10.0 * Tb * x->N * M * (x->cfg.causal ? 0.5 : 1.0);
    if (x->tok) {
      a0 = t0 / x->N * x->N; nseq = 1; p0 = t0 - a0; np = Tb;
      attn_flops = 10.0 * M * ((double)Tb * p0 + 0.5 * Tb * Tb);
      // the previous block's attention backward of this sequence's earlier chunks read
      // these dctx / D rows (same stack or capture only: otherwise already ordered)
      const unsigned long long cid = capture_id(sc);
      for (int64_t q = a0 / Tb; q < ai; ++q)
        if (x->atb_rec[q] && x->atb_cap[q] == cid && x->lanes[q % nl] != sc)
          FM_CUDA(cudaStreamWaitEvent(sc, x->ev_atb[q], 0));
    }
    GemmArgs g;
    g.M = (int)Tb; g.N = (int)M; g.K = (int)M;
    g.A = dA; g.lda = M; g.B = p->wo; g.ldb = M; g.b_kmajor = 1; g.C = dctx; g.ldc = M;
    FM_GEMM(KK_DCTX, g);
    if (x->tok) {  // dK/dV of this chunk's keys take the later chunks' queries (their dctx)
      FM_CUDA(cudaEventRecord(x->ev_dctx[ai], sc));
      for (int64_t q = ai + 1; q < (a0 + x->N) / Tb; ++q)
        if (x->lanes[q % nl] != sc) FM_CUDA(cudaStreamWaitEvent(sc, x->ev_dctx[q], 0));
    }
    FM_KP(KK_ATTN_B, attn_tc_supported(dt, (int)M, (int)x->H) ? 1 : 3, attn_flops, (double)Tb * 8 * M * es, sc,
          attn_bwd(dt, at<char>(saved, L.qkv + a0 * 3 * M * es), at<char>(saved, L.ctx + a0 * M * es),
                   at<float>(saved, L.lse + a0 * x->H * 4), (char*)x->dctx + a0 * M * es,
                   (char*)x->dqkv + a0 * 3 * M * es, x->Dbuf + a0 * x->H, (int)nseq, (int)x->N, (int)p0, (int)np,
                   (int)M, (int)x->H, x->cfg.causal, sc));
    if (x->tok) {
      FM_CUDA(cudaEventRecord(x->ev_atb[ai], sc));
      x->atb_rec[ai] = 1;
      x->atb_cap[ai] = capture_id(sc);
    }
    if (dx) {
      g = GemmArgs();
      g.M = (int)Tb; g.N = (int)M; g.K = (int)(3 * M);
      g.A = dqkv; g.lda = 3 * M; g.B = p->wqkv; g.ldb = 3 * M; g.b_kmajor = 1;
      g.C = (char*)dx + t0 * M * es; g.ldc = M;
      if (x->cfg.residual) { g.resid = dA; g.ldr = M; }
      FM_GEMM(KK_DX, g);
    }
    task_end(x, tk_atb, TK_ATB, x->at_split ? ai : -1, sc);
  }
  // ---- deferred MHA/gate wgrads over all T tokens (one K=T GEMM each), in the order
  // Wg, Wo (AR of [dWo|dWg] released), then Wqkv (AR of dWqkv released).
  cudaStream_t sc = nl > 1 ? x->s_wg : x->lanes[0];
  if (flowmoe_status st = join_lanes(x, sc)) return st;
  const int tk_wga = task_begin(x, sc);
  float* gf = gr->grad_flat;
  FM_KP(KK_DWG, 2, 2.0 * x->T * M * E, (double)x->T * M * es + x->T * E * 4.0 + M * E * 8.0, sc,
        gate_wgrad(dt, at<char>(saved, L.a), x->dl, gf + 4 * M * M, x->wg_part, (int)x->T, (int)M, (int)E, gacc, sc));
  GemmArgs g;
  g.M = (int)M; g.N = (int)M; g.K = (int)x->T;
  g.A = at<char>(saved, L.ctx); g.lda = M; g.a_mmajor = 1;
  g.B = x->dA; g.ldb = M;
  g.C = gf + 3 * M * M; g.ldc = M; g.epi = gepi;
  FM_GEMM(KK_DWO, g);
  FM_CUDA(cudaEventRecord(x->ev_grads_a, sc));
  g = GemmArgs();
  g.M = (int)M; g.N = (int)(3 * M); g.K = (int)x->T;
  g.A = xin; g.lda = M; g.a_mmajor = 1;
  g.B = x->dqkv; g.ldb = 3 * M;
  g.C = gf; g.ldc = 3 * M; g.epi = gepi;
  FM_GEMM(KK_DWQKV, g);
  task_end(x, tk_wga, TK_WGA, -1, sc);
  FM_CUDA(cudaEventRecord(x->ev_grads_b, sc));
  // ---- AR of the replicated grads, low priority, chunked by S_p (Alg. 2); centralized
  // policies defer every block's AR until the backward pass is over (allreduce_wait).
  FM_CUDA(cudaEventRecord(x->ev_bwd_done, sc));
  if (x->ev_wg_done[1]) {
    FM_CUDA(cudaEventRecord(x->ev_wg_done[wset], sc));
    x->wg_recorded[wset] = true;
    x->wg_cap_id[wset] = capture_id(sc);
  }
  // dx is ready once the lanes are done; with a separate wgrad stream the caller does
  // not wait for the wgrads (they finish under the next block's backward, and every
  // AR ticket / allreduce_wait orders after them)
  if (join) {
    if (sc != x->lanes[0]) {
      if (flowmoe_status st = join_lanes(x, x->lanes[0])) return st;
      FM_CUDA(cudaEventRecord(x->ev_done, x->lanes[0]));
    } else {
      FM_CUDA(cudaEventRecord(x->ev_done, sc));
    }
  }
  if (x->ar_pipelined) {
    if (flowmoe_status s = submit_ar(x, gf + 3 * M * M, (size_t)(M * M + M * E), chunk_bytes, x->ev_grads_a)) return s;
    if (flowmoe_status s = submit_ar(x, gf, (size_t)(3 * M * M), chunk_bytes, x->ev_grads_b)) return s;
    if (flowmoe_status s = new_ticket(x, ar)) return s;
  } else {
    const uint64_t t = x->next_ticket++;
    x->pending_ar.push_back({gf, (size_t)(4 * M * M + M * E), t});
    if (ar) *ar = t;
  }
  if (join) FM_CUDA(cudaStreamWaitEvent(stream, x->ev_done, 0));
  return FLOWMOE_OK;
}
}  // namespace

extern "C" {

flowmoe_status flowmoe_block_fwd(flowmoe_ctx* x, const flowmoe_params* p, const void* xin,
                                 void* y, void* saved, cudaStream_t stream) {
  apply_ctx(x);
  return enqueue_fwd(x, p, xin, y, saved, stream, true, true);
}

flowmoe_status flowmoe_block_bwd(flowmoe_ctx* x, const flowmoe_params* p, const void* xin,
                                 const void* saved, const void* dy, void* dx,
                                 const flowmoe_grads* gr, size_t chunk_bytes, flowmoe_ticket* ar,
                                 cudaStream_t stream) {
  apply_ctx(x);
  return enqueue_bwd(x, p, xin, saved, dy, dx, gr, chunk_bytes, ar, stream, true, true);
}

flowmoe_status flowmoe_stack_fwd(flowmoe_ctx* x, int L, const flowmoe_params* params, const void* x0,
                                 void* const* ys, void* const* saved, cudaStream_t stream) {
  apply_ctx(x);
  if (!x || L < 1 || !params || !x0 || !ys || !saved) return fail(FLOWMOE_ERR_INVALID, "stack_fwd: bad argument");
  for (int l = 0; l < L; ++l)
    if (flowmoe_status s = enqueue_fwd(x, &params[l], l ? ys[l - 1] : x0, ys[l], saved[l], stream, l == 0,
                                       l == L - 1))
      return s;
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_stack_bwd(flowmoe_ctx* x, int L, const flowmoe_params* params, const void* x0,
                                 void* const* ys, void* const* saved, const void* dy, void* const* dxs,
                                 const flowmoe_grads* grads, size_t chunk_bytes, flowmoe_ticket* tickets,
                                 cudaStream_t stream) {
  apply_ctx(x);
  if (!x || L < 1 || !params || !x0 || !ys || !saved || !dy || !dxs || !grads)
    return fail(FLOWMOE_ERR_INVALID, "stack_bwd: bad argument");
  for (int l = L - 1; l >= 0; --l)
    if (flowmoe_status s = enqueue_bwd(x, &params[l], l ? ys[l - 1] : x0, saved[l], l == L - 1 ? dy : dxs[l + 1],
                                       dxs[l], &grads[l], chunk_bytes, tickets ? &tickets[l] : nullptr, stream,
                                       l == L - 1, l == 0))
      return s;
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_allreduce_submit(flowmoe_ctx* x, float* buf, size_t count,
                                        size_t chunk_bytes, int priority, cudaEvent_t ready,
                                        flowmoe_ticket* out) {
  apply_ctx(x);
  if (!x || (!buf && count)) return fail(FLOWMOE_ERR_INVALID, "allreduce_submit: NULL argument");
  if (priority < 1) return fail(FLOWMOE_ERR_INVALID, "allreduce_submit: priority must be >= 1 (0 is A2A)");
  if (chunk_bytes == 0 || chunk_bytes % 16)
    return fail(FLOWMOE_ERR_INVALID, "allreduce_submit: chunk_bytes must be a positive multiple of 16");
  if (!ready) {
    if (flowmoe_status st = join_lanes(x, x->s_comp)) return st;
    FM_CUDA(cudaEventRecord(x->ev_grads_a, x->s_comp));
    ready = x->ev_grads_a;
  }
  if (flowmoe_status s = submit_ar(x, buf, count, chunk_bytes, ready)) return s;
  return new_ticket(x, out);
}

static flowmoe_status check_opt(const flowmoe_optimizer* o, int64_t step) {
  if (!o) return fail(FLOWMOE_ERR_INVALID, "optimizer is NULL");
  if (o->kind != FLOWMOE_OPT_SGD && o->kind != FLOWMOE_OPT_ADAMW)
    return fail(FLOWMOE_ERR_INVALID, "optimizer.kind must be FLOWMOE_OPT_SGD or FLOWMOE_OPT_ADAMW");
  if (!(o->lr >= 0.f) || !(o->weight_decay >= 0.f) || !(o->beta1 >= 0.f && o->beta1 < 1.f))
    return fail(FLOWMOE_ERR_INVALID, "optimizer: need lr >= 0, weight_decay >= 0, 0 <= beta1 < 1");
  if (o->kind == FLOWMOE_OPT_ADAMW && (!(o->beta2 >= 0.f && o->beta2 < 1.f) || !(o->eps >= 0.f)))
    return fail(FLOWMOE_ERR_INVALID, "optimizer: AdamW needs 0 <= beta2 < 1 and eps >= 0");
  if (step < 1) return fail(FLOWMOE_ERR_INVALID, "optimizer: step must be >= 1");
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_optimizer_step(flowmoe_ctx* x, const flowmoe_optimizer* o, int64_t step, float* master,
                                      float* s1, float* s2, const float* grad, void* weight, size_t n,
                                      cudaStream_t stream) {
  apply_ctx(x);
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (flowmoe_status st = check_opt(o, step)) return st;
  if (n == 0) return FLOWMOE_OK;
  if (!master || !s1 || !grad || (o->kind == FLOWMOE_OPT_ADAMW && !s2))
    return fail(FLOWMOE_ERR_INVALID, "optimizer_step: NULL tensor");
  FM_K(1, optim_step(x->dt, o->kind, o->lr, o->beta1, o->beta2, o->eps, o->weight_decay, step, master, s1, s2,
                     grad, weight, (int64_t)n, stream));
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_embed_fwd(flowmoe_ctx* x, const void* table, int64_t V, const int32_t* ids, int64_t T,
                                 void* out, cudaStream_t stream) {
  apply_ctx(x);
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (T < 0 || V < 1) return fail(FLOWMOE_ERR_INVALID, "embed_fwd: need T >= 0 and V >= 1");
  if (T == 0) return FLOWMOE_OK;
  if (!table || !ids || !out) return fail(FLOWMOE_ERR_INVALID, "embed_fwd: NULL pointer");
  FM_K(1, embed_fwd(x->dt, table, ids, out, T, V, (int)x->M, stream));
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_embed_bwd(flowmoe_ctx* x, const int32_t* ids, int64_t T, const void* dx, int64_t V,
                                 float* dtable, cudaStream_t stream) {
  apply_ctx(x);
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (T < 0 || V < 1) return fail(FLOWMOE_ERR_INVALID, "embed_bwd: need T >= 0 and V >= 1");
  if (T == 0) return FLOWMOE_OK;
  if (!ids || !dx || !dtable) return fail(FLOWMOE_ERR_INVALID, "embed_bwd: NULL pointer");
  FM_K(1, embed_bwd(x->dt, ids, dx, dtable, T, V, (int)x->M, stream));
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_xent(flowmoe_ctx* x, const float* logits, const int32_t* labels, int64_t T, int64_t V,
                            float scale, float* losses, float* loss, void* dlogits, cudaStream_t stream) {
  apply_ctx(x);
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (T < 0 || V < 1) return fail(FLOWMOE_ERR_INVALID, "xent: need T >= 0 and V >= 1");
  if (T > 0 && (!logits || !labels || !losses)) return fail(FLOWMOE_ERR_INVALID, "xent: NULL logits/labels/losses");
  FM_K(T > 0 ? 1 + (loss ? 1 : 0) : 0, xent(x->dt, logits, labels, T, V, scale, losses, loss, dlogits, stream));
  return FLOWMOE_OK;
}

static flowmoe_status check_lm(const flowmoe_ctx* x, int64_t T, int64_t V) {
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (T < 0 || V < 8 || V % 8 != 0 || T > INT32_MAX || V > INT32_MAX)
    return fail(FLOWMOE_ERR_INVALID, "lm_head: need 0 <= T < 2^31 and V a positive multiple of 8 (< 2^31)");
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_lm_head_fwd(flowmoe_ctx* x, const void* h, const void* w, int64_t T, int64_t V, float* logits,
                                   cudaStream_t stream) {
  apply_ctx(x);
  if (flowmoe_status st = check_lm(x, T, V)) return st;
  if (T == 0) return FLOWMOE_OK;
  if (!h || !w || !logits) return fail(FLOWMOE_ERR_INVALID, "lm_head_fwd: NULL pointer");
  GemmArgs g;  // logits[T][V] = h[T][M] · W[V][M]ᵀ (W is K-major for this product)
  g.M = (int)T; g.N = (int)V; g.K = (int)x->M;
  g.A = h; g.lda = x->M;
  g.B = w; g.ldb = x->M; g.b_kmajor = 1;
  g.C = logits; g.ldc = V; g.epi = EPI_STORE_F32;
  FM_K(1, gemm(g, x->dt, stream));
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_lm_head_bwd(flowmoe_ctx* x, const void* h, const void* w, const void* dlogits, int64_t T,
                                   int64_t V, void* dh, float* dw, cudaStream_t stream) {
  apply_ctx(x);
  if (flowmoe_status st = check_lm(x, T, V)) return st;
  if (T == 0) return FLOWMOE_OK;
  if (!dlogits || (dh && !w) || (dw && !h)) return fail(FLOWMOE_ERR_INVALID, "lm_head_bwd: NULL pointer");
  if (dh) {
    GemmArgs g;  // dh[T][M] = dlogits[T][V] · W[V][M]
    g.M = (int)T; g.N = (int)x->M; g.K = (int)V;
    g.A = dlogits; g.lda = V;
    g.B = w; g.ldb = x->M;
    g.C = dh; g.ldc = x->M; g.epi = EPI_STORE;
    FM_K(1, gemm(g, x->dt, stream));
  }
  if (dw) {
    GemmArgs g;  // dW[V][M] += dlogitsᵀ · h  (dlogits is M-major for this product)
    g.M = (int)V; g.N = (int)x->M; g.K = (int)T;
    g.A = dlogits; g.lda = V; g.a_mmajor = 1;
    g.B = h; g.ldb = x->M;
    g.C = dw; g.ldc = x->M; g.epi = EPI_ACC_F32;
    FM_K(1, gemm(g, x->dt, stream));
  }
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_expert_update(flowmoe_ctx* x, const flowmoe_optimizer* o, int64_t step,
                                     const flowmoe_expert_opt* st, const flowmoe_grads* gr, flowmoe_ticket* done) {
  apply_ctx(x);
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (flowmoe_status s = check_opt(o, step)) return s;
  if (!st || !gr || !gr->dw1 || !gr->db1 || !gr->dw2 || !gr->db2)
    return fail(FLOWMOE_ERR_INVALID, "expert_update: NULL argument");
  const float* g[4] = {gr->dw1, gr->db1, gr->dw2, gr->db2};
  const int64_t n[4] = {x->El * x->M * x->F, x->El * x->F, x->El * x->F * x->M, x->El * x->M};
  for (int i = 0; i < 4; ++i)
    if (!st->master[i] || !st->state1[i] || (o->kind == FLOWMOE_OPT_ADAMW && !st->state2[i]))
      return fail(FLOWMOE_ERR_INVALID, "expert_update: NULL optimizer tensor");
  // behind the latest block's expert wgrads on the weight-gradient stream (in order)
  cudaStream_t sw = x->s_wg;
  for (int i = 0; i < 4; ++i)
    FM_K(1, optim_step(x->dt, o->kind, o->lr, o->beta1, o->beta2, o->eps, o->weight_decay, step, st->master[i],
                       st->state1[i], st->state2[i], g[i], st->weight[i], n[i], sw));
  // a ticket like the all-reduce's: flowmoe_allreduce_wait(done) orders a stream after it
  const uint64_t t = x->next_ticket++;
  FM_CUDA(cudaEventRecord(x->ticket_ev[t % NUM_TICKET_EVENTS], sw));
  if (done) *done = t;
  return FLOWMOE_OK;
}

flowmoe_status flowmoe_allreduce_wait(flowmoe_ctx* x, flowmoe_ticket t, cudaStream_t stream) {
  apply_ctx(x);
  if (!x) return fail(FLOWMOE_ERR_INVALID, "ctx is NULL");
  if (t == 0 || t >= x->next_ticket || x->next_ticket - t > NUM_TICKET_EVENTS)
    return fail(FLOWMOE_ERR_STATE, "allreduce_wait: unknown or expired ticket");
  if (x->P > 1 && !x->group) {
    ncclResult_t a = ncclSuccess, b = ncclSuccess;
    for (ncclComm_t c : x->a2a_comm) {
      ncclResult_t e = ncclSuccess;
      ncclCommGetAsyncError(c, &e);
      if (e != ncclSuccess) a = e;
    }
    if (x->comm_ar) ncclCommGetAsyncError(x->comm_ar, &b);
    if (a != ncclSuccess || b != ncclSuccess)
      return fail(FLOWMOE_ERR_NCCL, std::string("async NCCL error: ") + ncclGetErrorString(a != ncclSuccess ? a : b));
  }
  if (LocalGroup* g = x->group) {
    std::lock_guard<std::mutex> lk(g->mu);
    const int rk = x->cfg.rank;
    if (g->ticket_sub[rk].count(t) && !g->ticket_done[rk].count(t))
      return fail(FLOWMOE_ERR_STATE, "allreduce_wait: the other ranks of the local group have not submitted "
                                     "their matching all-reduce yet");
  }
  if (!x->pending_ar.empty()) {
    // centralized AR: every pending block AR, whole tensors, after the last backward
    FM_CUDA(cudaStreamWaitEvent(x->s_ar, x->ev_bwd_done, 0));
    for (const auto& pa : x->pending_ar)
      if (flowmoe_status s = submit_ar(x, pa.buf, pa.count, pa.count * 4, nullptr)) return s;
    for (const auto& pa : x->pending_ar)
      FM_CUDA(cudaEventRecord(x->ticket_ev[pa.ticket % NUM_TICKET_EVENTS], x->s_ar));
    x->pending_ar.clear();
  }
  FM_CUDA(cudaStreamWaitEvent(stream, x->ticket_ev[t % NUM_TICKET_EVENTS], 0));
  return FLOWMOE_OK;
}

void flowmoe_destroy(flowmoe_ctx* x) {
  if (!x) return;
  LocalGroup* g = x->group;
  if (g) {  // peers may still be exchanging with this member: drain the device first
    cudaDeviceSynchronize();
    g->m[x->cfg.rank] = nullptr;
    bool last = true;
    for (flowmoe_ctx* m : g->m) last = last && !m;
    if (last) {
      if (g->s) cudaStreamDestroy(g->s);
      for (auto e : g->ev_pool) cudaEventDestroy(e);
      delete g;
    }
    x->group = nullptr;
  }
  for (size_t l = 1; l < x->lanes.size(); ++l) cudaStreamSynchronize(x->lanes[l]);
  if (x->s_wg && x->s_wg != x->s_comp) cudaStreamSynchronize(x->s_wg);
  if (x->s_comp) cudaStreamSynchronize(x->s_comp);
  if (x->s_a2a) cudaStreamSynchronize(x->s_a2a);
  if (x->s_ar) cudaStreamSynchronize(x->s_ar);
  for (size_t l = 1; l < x->a2a_stream.size(); ++l) cudaStreamSynchronize(x->a2a_stream[l]);
  for (size_t l = 1; l < x->a2a_comm.size(); ++l) ncclCommDestroy(x->a2a_comm[l]);
  for (size_t l = 1; l < x->a2a_stream.size(); ++l) cudaStreamDestroy(x->a2a_stream[l]);
  if (x->comm_ar) ncclCommDestroy(x->comm_ar);
  if (x->comm_a2a) ncclCommDestroy(x->comm_a2a);
  for (auto* v : {&x->ev_at, &x->ev_d, &x->ev_e, &x->ev_c, &x->ev_cb, &x->ev_cba, &x->ev_eb, &x->ev_dba,
                  &x->ev_qkv, &x->ev_dctx, &x->ev_atb})
    for (auto e : *v) if (e) cudaEventDestroy(e);
  for (auto e : x->ticket_ev) if (e) cudaEventDestroy(e);
  for (auto e : x->ev_sent) if (e) cudaEventDestroy(e);
  for (auto e : x->ev_lane) if (e) cudaEventDestroy(e);
  for (auto e : x->ev_wg_done) if (e) cudaEventDestroy(e);
  for (size_t l = 1; l < x->lanes.size(); ++l) cudaStreamDestroy(x->lanes[l]);
  if (x->s_wg && x->s_wg != x->s_comp) cudaStreamDestroy(x->s_wg);
  for (auto e : {x->ev_in, x->ev_done, x->ev_grads_a, x->ev_grads_b, x->ev_bwd_done}) if (e) cudaEventDestroy(e);
  for (void* p : x->ipc_opened) cudaIpcCloseMemHandle(p);
  for (auto e : x->prof.pool) cudaEventDestroy(e);
  for (auto e : x->tlog.pool) cudaEventDestroy(e);
  if (x->tlog.base) cudaEventDestroy(x->tlog.base);
  if (g_prof == &x->prof) g_prof = nullptr;
  for (void* p : x->allocs) cudaFree(p);
  if (x->sk_test_ws) cudaFree(x->sk_test_ws);
  if (x->sk_test_tick) cudaFree(x->sk_test_tick);
  if (x->s_comp) cudaStreamDestroy(x->s_comp);
  if (x->s_a2a) cudaStreamDestroy(x->s_a2a);
  if (x->s_ar) cudaStreamDestroy(x->s_ar);
  delete x;
}

}  // extern "C"

extern "C" flowmoe_status flowmoe_test_gemm(flowmoe_ctx* x, int dtype, int M, int N, int K, int batch,
                                            const void* A, int64_t lda, int64_t sA, int a_mmajor,
                                            const void* B, int64_t ldb, int64_t sB, int b_kmajor,
                                            void* C, int64_t ldc, int64_t sC, int epi,
                                            const void* bias, const void* resid, void* aux,
                                            cudaStream_t stream) {
  GemmArgs g;
  g.M = M; g.N = N; g.K = K; g.batch = batch;
  g.A = A; g.lda = lda; g.sA = sA; g.a_mmajor = a_mmajor;
  g.B = B; g.ldb = ldb; g.sB = sB; g.b_kmajor = b_kmajor;
  g.C = C; g.ldc = ldc; g.sC = sC; g.epi = epi;
  g.bias = bias; g.sBias = N;
  g.resid = resid; g.ldr = ldc; g.sR = sC;
  g.aux = aux; g.ldaux = ldc; g.sAux = sC;
  if (dtype != DT_F32 && dtype != DT_BF16) return fail(FLOWMOE_ERR_INVALID, "dtype");
  if (x) {
    apply_ctx(x);
    if (dtype == DT_BF16) {
      if (!x->sk_test_ws) {
        if (cudaMalloc((void**)&x->sk_test_ws, SK_WS_FLOATS * 4) != cudaSuccess ||
            cudaMalloc((void**)&x->sk_test_tick, SK_TICKS * 4) != cudaSuccess ||
            cudaMemset(x->sk_test_tick, 0, SK_TICKS * 4) != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess)
          return fail(FLOWMOE_ERR_OOM, "stream-K scratch");
      }
      g.splitk_ws = x->sk_test_ws; g.splitk_ws_floats = SK_WS_FLOATS;
      g.splitk_tick = x->sk_test_tick; g.splitk_ticks = SK_TICKS;
    }
  } else {  // library defaults, no profile
    gemm_tc_set_debug(0);
    gemm_tc_force_bn(0);
    gemm_tc_force_cg(0);
    gemm_tc_force_streamk(0);
    g_pdl_enabled = 1;
    g_prof = nullptr;
  }
  FM_KP(KK_TEST, 1, 2.0 * M * N * (double)K * batch, 0, stream, gemm(g, dtype, stream));
  return FLOWMOE_OK;
}
