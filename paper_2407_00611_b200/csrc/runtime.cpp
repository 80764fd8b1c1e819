// runtime.cpp -- the C ABI of include/wf.h: context, workspace, and the WallFacer
// schedule (forward: Alg. 1; backward: PAPER.md:201-205) driving the
// sm_100a block kernels and the NVLink peer-memory transport (copy-engine pushes into the
// peers' CUDA-IPC-mapped workspaces, release/acquire flags).
//
// One schedule implementation serves three modes:
//   real      : one process per GPU (or, for tests, several processes sharing one GPU);
//               this rank executes its pushes, waits and block kernels; records its sends.
//               Bootstrap (the IPC handle exchange) through NCCL (wf_init) or a caller
//               supplied host all-gather (wf_init_bootstrap).
//   emulated  : all P ranks on this GPU; every message is a device-local copy.
//   dry       : no GPU work at all; only the CommTrace is produced (wf_plan_trace).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/wf.h"
#include "common.h"
#include "internal.h"
#include "plan.h"

namespace wf {
namespace {

typedef __nv_bfloat16 bf16;

struct Geo {
  int P, C, T, R, W;
  bool paper, causal;
  bool direct;        // DIRECT-PULL init (paper regime): K/V units straight from their owners
  int64_t N;
  int n, c, h, d;     // n rows per rank; c = chunk rows for position tables
  int64_t E;          // h * d
  int Bk;             // rows of the K/V block a rank attends per step (C*n paper, W*n ext)
};

// Per-rank device workspace (one set per virtual rank in emulated mode).
struct RankBufs {
  // forward
  bf16 *qt = nullptr, *kt = nullptr, *vt = nullptr;  // team Q/K/V (C*n rows)
  bf16 *rk[2] = {nullptr, nullptr}, *rv[2] = {nullptr, nullptr};  // ring / slice K,V (Bk rows)
  float *o_state = nullptr, *lse_state = nullptr;    // fp32 (C*n rows), lse [C][h][n]
  float* rs_o = nullptr;                             // [C][n rows] fp32 partials of my rows
  float* rs_lse = nullptr;                           // [C][h][n]
  // backward
  float* dsum = nullptr;                             // [h][n] -D / sqrt(d) of my rows
  float* nlse = nullptr;                             // [h][n] -LSE log2(e) of my rows
  bf16* t_do = nullptr;                              // team dO (C*n rows)
  float *t_lse = nullptr, *t_dsum = nullptr;         // [C][h][n]
  bf16 *pq[2] = {nullptr, nullptr}, *pdo[2] = {nullptr, nullptr};
  float *plse[2] = {nullptr, nullptr}, *pdsum[2] = {nullptr, nullptr}, *pdq[2] = {nullptr, nullptr};
  float* home_dq = nullptr;                          // C*n rows fp32
  float *dk_acc = nullptr, *dv_acc = nullptr;        // Bk rows fp32
  float *rev_k = nullptr, *rev_v = nullptr;          // paper: C*n rows; ext: [T][n rows]
  float *rsq = nullptr, *rsk = nullptr, *rsv = nullptr;  // [C][n rows]
};

struct Seg {
  const void* src;
  void* dst;
  int64_t bytes;
};

struct Xfer {
  int pass, kind, step, src, dst, block;
  std::vector<Seg> segs;
  bool pull = false;   // peer-memory transport: the consumer kernel reads the source in place
  bool fused = false;  // already delivered by a producer kernel's epilogue (wf_qkv_proj)
};

constexpr size_t kFlagBytes = 4096;  // flag block at the start of every rank's workspace
constexpr int kMaxRanks = 64;

}  // namespace
}  // namespace wf

using namespace wf;

struct wf_ctx {
  Plan plan;
  int rank = 0;
  bool emulated = false, dry = false;
  int dry_rank = -1;  // dry mode: record only events touching this rank as sender (-1: all)
  ncclComm_t comm = nullptr;                      // bootstrap only (wf_init)
  wf_allgather_fn ag_fn = nullptr;                // bootstrap only (wf_init_bootstrap)
  void* ag_user = nullptr;
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  // workspace
  int64_t ws_key[5] = {0, 0, 0, 0, 0};
  void* ws = nullptr;
  size_t ws_bytes = 0;
  std::vector<RankBufs> rb;
  std::vector<wf_event> trace_fwd, trace_bwd;
  int64_t launches = 0;
  std::string err;
  int debug = 0;
  int sched = WF_SCHED_GATHER_SHUFFLE;  // wf_set_schedule
  // set by wf_qkv_proj when its epilogue already delivered the team gather of (Q, K, V);
  // consumed only by the wf_attn_fwd that immediately follows it on this context (call
  // sequence numbers), with the same tensors and geometry
  const void *proj_q = nullptr, *proj_k = nullptr, *proj_v = nullptr;
  int64_t proj_key[4] = {0, 0, 0, 0};
  uint64_t seq = 0, proj_seq = 0;
  // asynchronous failure reporting (WF_ERR_COMM): a wait that times out writes these
  // host-mapped words ([0] = 1, [1] = expected count, [2] = count seen) instead of trapping
  volatile uint32_t* hfail = nullptr;
  uint32_t* dfail = nullptr;
  uint64_t timeout_ns = 30000000000ull;
  // WF_DEBUG_CHECKS builds: the memory ranges a call may touch (caller tensors + workspaces)
  std::vector<std::pair<const char*, size_t>> dbg_ranges;
  // peer-memory transport (real mode, P > 1): CUDA IPC mapped workspaces + flag signalling
  bool ipc = false;
  std::vector<char*> peer_base;
  std::vector<RankBufs> rbp;       // my layout translated into each rank's address space
  uint32_t sent[2][kMaxRanks] = {}, rcvd[2][kMaxRanks] = {};
  uint32_t acks_sent[kMaxRanks] = {}, ack_base[kMaxRanks] = {};  // monotonic across calls
  uint32_t epoch = 0;
  std::vector<cudaEvent_t> ev_step, ev_src;
  cudaEvent_t ev_c = nullptr;
  // kernel timing (bench)
  bool profiling = false;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_fwd, ev_bwd;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> ev_phase;  // (kind, events)
  std::vector<cudaEvent_t> ev_pool;
};

namespace {

thread_local std::string g_ctxless_err;

wf_status fail(wf_ctx* c, wf_status s, const std::string& msg) {
  if (c)
    c->err = msg;
  else
    g_ctxless_err = msg;
  return s;
}

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return fail(ctx, WF_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define NCK(x)                                                                                   \
  do {                                                                                           \
    ncclResult_t r_ = (x);                                                                       \
    if (r_ != ncclSuccess) return fail(ctx, WF_ERR_COMM, std::string(#x ": ") + ncclGetErrorString(r_)); \
  } while (0)
#define WCK(x)                      \
  do {                              \
    wf_status s_ = (x);             \
    if (s_ != WF_OK) return s_;     \
  } while (0)

bool local(const wf_ctx* ctx, int r) { return ctx->emulated || (!ctx->dry && r == ctx->rank); }
bool recorded(const wf_ctx* ctx, int src) {
  if (ctx->dry) return ctx->dry_rank < 0 || src == ctx->dry_rank;
  return ctx->emulated || src == ctx->rank;
}

wf_status check_shape(wf_ctx* ctx, int64_t N, int heads, int head_dim, int causal, Geo* g) {
  const Plan& p = ctx->plan;
  if (head_dim != 64 && head_dim != 72 && head_dim != 128)
    return fail(ctx, WF_ERR_CONFIG, "head_dim must be 64, 72 or 128");
  if (heads < 1) return fail(ctx, WF_ERR_CONFIG, "heads must be >= 1");
  const int64_t q = causal ? 2LL * p.P * WF_TILE : static_cast<int64_t>(p.P) * WF_TILE;
  if (N <= 0 || N % q) return fail(ctx, WF_ERR_CONFIG, "N must be a positive multiple of " + std::to_string(q));
  if (N / p.P > (1LL << 30) / 2) return fail(ctx, WF_ERR_CONFIG, "N/P too large");
  g->P = p.P;
  g->C = p.C;
  g->T = p.T;
  g->R = p.R;
  g->W = p.W;
  g->paper = p.paper;
  g->direct = ctx->sched == WF_SCHED_DIRECT_PULL && p.paper && p.C > 1;
  g->causal = causal != 0;
  g->N = N;
  g->n = static_cast<int>(N / p.P);
  g->c = causal ? static_cast<int>(N / (2 * p.P)) : g->n;
  g->h = heads;
  g->d = head_dim;
  g->E = static_cast<int64_t>(heads) * head_dim;
  g->Bk = p.paper ? p.C * g->n : p.W * g->n;
  if (p.C > WF_MAX_PARTS || (!p.paper && p.T > WF_MAX_PARTS) || 2 * std::max(p.C, p.W) > WF_MAX_CHUNKS)
    return fail(ctx, WF_ERR_CONFIG, "P/C too large for this build");
  return WF_OK;
}

// Chunk position table of a list of units (zigzag: two chunks per unit).
PosTable units_table(const Geo& g, int u0, int count) {
  PosTable t;
  std::memset(&t, 0, sizeof(t));
  t.chunk = g.c;
  int k = 0;
  for (int u = u0; u < u0 + count; ++u) {
    if (g.causal) {
      t.start[k++] = u * g.c;
      t.start[k++] = (2 * g.P - 1 - u) * g.c;
    } else {
      t.start[k++] = u * g.n;
    }
  }
  t.nchunks = k;
  t.tpc_shift = tpc_shift_of(t.chunk);
  return t;
}

// ------------------------------------------------------------------ peer memory
// Exchange CUDA IPC handles of every rank's workspace (an NCCL all-gather of the 64-byte
// handles), map the peers' workspaces, and translate my buffer layout into each rank's
// address space (all ranks carve identical layouts).
RankBufs translate(const RankBufs& b, const char* from, const char* to) {
  RankBufs t = b;
  char** f = reinterpret_cast<char**>(&t);
  for (size_t i = 0; i < sizeof(RankBufs) / sizeof(char*); ++i)
    if (f[i]) f[i] = const_cast<char*>(to) + (f[i] - from);
  return t;
}

// Bootstrap all-gather of `bytes` host bytes per rank (rank-major into out): the caller's
// host collective (wf_init_bootstrap) or NCCL over the bootstrap communicator (wf_init).
wf_status boot_allgather(wf_ctx* ctx, const void* in, void* out, size_t bytes) {
  const int P = ctx->plan.P, me = ctx->rank;
  if (ctx->ag_fn) {
    if (ctx->ag_fn(in, out, bytes, ctx->ag_user) != 0) return fail(ctx, WF_ERR_COMM, "bootstrap all-gather failed");
    return WF_OK;
  }
  if (!ctx->comm) return fail(ctx, WF_ERR_COMM, "no bootstrap communicator");
  void* dbuf = nullptr;
  CK(cudaMalloc(&dbuf, static_cast<size_t>(P) * bytes));
  CK(cudaMemcpy(static_cast<char*>(dbuf) + me * bytes, in, bytes, cudaMemcpyHostToDevice));
  NCK(ncclAllGather(static_cast<char*>(dbuf) + me * bytes, dbuf, bytes, ncclInt8, ctx->comm, ctx->comm_stream));
  CK(cudaStreamSynchronize(ctx->comm_stream));
  CK(cudaMemcpy(out, dbuf, P * bytes, cudaMemcpyDeviceToHost));
  CK(cudaFree(dbuf));
  return WF_OK;
}

wf_status exchange_ipc(wf_ctx* ctx) {
  const int P = ctx->plan.P, me = ctx->rank;
  for (size_t r = 0; r < ctx->peer_base.size(); ++r)
    if (static_cast<int>(r) != me && ctx->peer_base[r]) cudaIpcCloseMemHandle(ctx->peer_base[r]);
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, ctx->ws));
  std::vector<cudaIpcMemHandle_t> hs(P);
  WCK(boot_allgather(ctx, &h, hs.data(), sizeof(h)));
  ctx->peer_base.assign(P, nullptr);
  ctx->rbp.assign(P, RankBufs{});
  for (int r = 0; r < P; ++r) {
    if (r == me) {
      ctx->peer_base[r] = static_cast<char*>(ctx->ws);
    } else {
      void* p = nullptr;
      CK(cudaIpcOpenMemHandle(&p, hs[r], cudaIpcMemLazyEnablePeerAccess));
      ctx->peer_base[r] = static_cast<char*>(p);
    }
    ctx->rbp[r] = translate(ctx->rb[0], static_cast<char*>(ctx->ws), ctx->peer_base[r]);
  }
  // fresh flag blocks everywhere: no stale counts
  std::memset(ctx->sent, 0, sizeof(ctx->sent));
  std::memset(ctx->rcvd, 0, sizeof(ctx->rcvd));
  std::memset(ctx->acks_sent, 0, sizeof(ctx->acks_sent));
  std::memset(ctx->ack_base, 0, sizeof(ctx->ack_base));
  ctx->epoch = 0;
  // every rank has zeroed its flags before anyone signals (the all-gather above ordered
  // the memsets; this second one orders the mappings)
  int32_t one = me;
  std::vector<int32_t> all(P);
  return boot_allgather(ctx, &one, all.data(), sizeof(one));
}

// flag addresses: data[chan][src] at word chan*64 + src, ack[src] at 128 + src, bar[src] at 192 + src
uint32_t* flag_of(wf_ctx* ctx, int owner, int word) {
  return reinterpret_cast<uint32_t*>(ctx->peer_base[owner]) + word;
}

wf_status ipc_barrier(wf_ctx* ctx, cudaStream_t st);

// ------------------------------------------------------------------ workspace
// The workspace carve of one rank (bytes per buffer, in carve order), sized by regime:
// only the buffers this (P, C, R) schedule touches.  `copies`: messages land in receive
// slots (emulated mode); with peer memory the reductions read the senders' partials in
// place, so the merge / dQ-sum / dK-dV replica slots exist only where partials are pushed
// (the unit-pipelined extension regime).
using CarveList = std::vector<std::pair<void**, int64_t>>;
void carve_rank(const Geo& g, RankBufs& b, CarveList& items, bool copies) {
  const int64_t C = g.C, n = g.n, E = g.E, h = g.h, Bk = g.Bk;
  const int64_t team = C * n * E;  // elements of a team tensor
  auto add = [&](auto** p, int64_t bytes) { items.push_back({reinterpret_cast<void**>(p), bytes}); };
  const bool pushed = copies || !g.paper;  // partials pushed into their owners' slots
  if (C > 1) {
    add(&b.qt, team * 2);
    add(&b.t_do, team * 2);
    add(&b.t_lse, C * h * n * 4);
    add(&b.t_dsum, C * h * n * 4);
    if (pushed) {
      add(&b.rs_o, team * 4);
      add(&b.rs_lse, C * h * n * 4);
      add(&b.rsq, team * 4);
    }
    if (g.paper && !g.direct) {
      add(&b.kt, team * 2);
      add(&b.vt, team * 2);
    }
  }
  // K/V receive slots: double-buffered ring (R > 1), one slot for the init block / slice
  // (R = 1, P > 1), none on one GPU (the caller's K/V are the whole sequence)
  const int kv_slots = g.R > 1 ? 2 : (g.P > 1 ? 1 : 0);
  for (int s = 0; s < kv_slots; ++s) {
    add(&b.rk[s], Bk * E * 2);
    add(&b.rv[s], Bk * E * 2);
  }
  if (g.P > 1) {  // one GPU writes the final bf16 output straight from the block kernel
    add(&b.o_state, team * 4);
    add(&b.lse_state, C * h * n * 4);
  }
  add(&b.dsum, h * n * 4);
  add(&b.nlse, h * n * 4);
  for (int s = 0; s < (g.R > 1 ? 2 : 1); ++s) {
    add(&b.pdq[s], team * 4);
    if (g.R > 1) {
      add(&b.pq[s], team * 2);
      add(&b.pdo[s], team * 2);
      add(&b.plse[s], C * h * n * 4);
      add(&b.pdsum[s], C * h * n * 4);
    }
  }
  if (g.R > 1) add(&b.home_dq, team * 4);
  if (g.P > 1) {  // one GPU writes bf16 dK/dV straight from the block kernel
    add(&b.dk_acc, Bk * E * 4);
    add(&b.dv_acc, Bk * E * 4);
  }
  if (copies) {  // dK/dV replica slots on the owner (holders of a unit: C paper, T extension)
    const int64_t slots = g.paper ? C : g.T;
    add(&b.rev_k, slots * n * E * 4);
    add(&b.rev_v, slots * n * E * 4);
  }
}

size_t carve_total(const CarveList& items) {
  size_t total = kFlagBytes;
  for (auto& it : items) total += (static_cast<size_t>(it.second) + 1023) & ~size_t(1023);
  return total;
}

wf_status ensure_ws(wf_ctx* ctx, const Geo& g) {
  if (ctx->dry) {
    ctx->rb.assign(ctx->plan.P, RankBufs{});
    return WF_OK;
  }
  const int64_t key[5] = {g.N, g.h, g.d, g.causal, g.direct};
  if (ctx->ws && std::equal(key, key + 5, ctx->ws_key)) return WF_OK;
  if (ctx->ws) {
    CK(cudaDeviceSynchronize());
    if (ctx->ipc) {
      // peers may still be reading (pull kernels) or signalling into this workspace from
      // their previous call: free it only after every rank has finished that call
      WCK(ipc_barrier(ctx, ctx->comm_stream));
      CK(cudaStreamSynchronize(ctx->comm_stream));
    }
    for (size_t r = 0; r < ctx->peer_base.size(); ++r)
      if (static_cast<int>(r) != ctx->rank && ctx->peer_base[r]) cudaIpcCloseMemHandle(ctx->peer_base[r]);
    ctx->peer_base.clear();
    CK(cudaFree(ctx->ws));
    ctx->ws = nullptr;
  }
  const int nranks = ctx->emulated ? g.P : 1;
  CarveList items;
  std::vector<RankBufs> rb(nranks);
  for (auto& b : rb) carve_rank(g, b, items, ctx->emulated);
  const size_t total = carve_total(items);
  void* base = nullptr;
  CK(cudaMalloc(&base, total));
  CK(cudaMemset(base, 0, kFlagBytes));
  CK(cudaDeviceSynchronize());
  size_t off = kFlagBytes;
  for (auto& it : items) {
    *it.first = static_cast<char*>(base) + off;
    off += (static_cast<size_t>(it.second) + 1023) & ~size_t(1023);
  }
  ctx->ws = base;
  ctx->ws_bytes = total;
  std::copy(key, key + 5, ctx->ws_key);
  ctx->rb = rb;
  if (ctx->ipc) WCK(exchange_ipc(ctx));
  return WF_OK;
}

RankBufs& B(wf_ctx* ctx, int r) {
  if (ctx->ipc && !ctx->dry) return ctx->rbp[r];
  return ctx->rb[ctx->emulated || ctx->dry ? r : 0];
}
// a rank's workspace buffer is addressable here: own/emulated ranks, or any rank with IPC
bool addressable(const wf_ctx* ctx, int r) { return local(ctx, r) || (ctx->ipc && !ctx->dry); }

cudaEvent_t pool_event(wf_ctx* ctx);
cudaEvent_t prof_begin(wf_ctx* ctx, cudaStream_t st);
wf_status dbg_check_segs(wf_ctx* ctx, const std::vector<Xfer>& xs);
wf_status dbg_check(wf_ctx* ctx, const void* p, int64_t bytes, const char* what);

// Launch a signal/wait kernel whose waits report a timeout through the context's
// host-mapped failure words (WF_ERR_COMM on the next call) instead of trapping.
wf_status sigwait(wf_ctx* ctx, SigArgs sig, SigArgs wt, cudaStream_t st) {
  wt.fail = ctx->dfail;
  wt.timeout_ns = ctx->timeout_ns;
  CK(launch_signal_wait(sig, wt, st));
  return WF_OK;
}

// ------------------------------------------------------------------ transport
// part: kPhaseAll, or (peer-memory transport) kPhaseSend = trace + copies + signals only and
// kPhaseWait = the matching waits only, so a sender can release a slot between the two.
enum { kPhaseAll = 0, kPhaseSend = 1, kPhaseWait = 2 };
wf_status run_phase(wf_ctx* ctx, std::vector<Xfer>& xs, std::vector<wf_event>& trace, cudaStream_t st,
                    int part = kPhaseAll) {
  if (part != kPhaseWait) {
    for (const Xfer& x : xs) {
      if (x.src == x.dst || !recorded(ctx, x.src)) continue;
      int64_t bytes = 0;
      for (const Seg& s : x.segs) bytes += s.bytes;
      trace.push_back(wf_event{x.pass, x.kind, x.step, x.src, x.dst, x.block, bytes});
    }
  }
  if (ctx->dry) return WF_OK;
  if (part != kPhaseWait) WCK(dbg_check_segs(ctx, xs));
  if (ctx->debug & WF_DEBUG_NO_TRANSFER) return WF_OK;
  if (ctx->emulated) {
    if (part == kPhaseWait) return WF_OK;
    for (const Xfer& x : xs)
      if (!x.fused)
        for (const Seg& s : x.segs)
        if (s.bytes && s.src != s.dst) CK(cudaMemcpyAsync(s.dst, s.src, s.bytes, cudaMemcpyDeviceToDevice, st));
    return WF_OK;
  }
  const int me = ctx->rank;
  const int ch = st == ctx->comm_stream ? 1 : 0;
  cudaEvent_t pe0 = xs.empty() ? nullptr : prof_begin(ctx, st);
  if (part != kPhaseWait) {
    for (const Xfer& x : xs) {
      if (x.src != me || x.pull || x.fused) continue;
      for (const Seg& sg : x.segs)
        if (sg.bytes && sg.src != sg.dst) CK(cudaMemcpyAsync(sg.dst, sg.src, sg.bytes, cudaMemcpyDefault, st));
    }
  }
  SigArgs sig{}, wt{};
  bool dst_done[kMaxRanks] = {}, src_done[kMaxRanks] = {};
  for (const Xfer& x : xs) {
    if (part != kPhaseWait && x.src == me && x.dst != me && !dst_done[x.dst]) {
      dst_done[x.dst] = true;
      sig.dst[sig.n] = flag_of(ctx, x.dst, ch * 64 + me);
      sig.val[sig.n++] = ++ctx->sent[ch][x.dst];
    }
    if (part != kPhaseSend && x.dst == me && x.src != me && !src_done[x.src]) {
      src_done[x.src] = true;
      wt.dst[wt.n] = flag_of(ctx, me, ch * 64 + x.src);
      wt.val[wt.n++] = ++ctx->rcvd[ch][x.src];
    }
  }
  WCK(sigwait(ctx, sig, wt, st));
  if (pe0) {
    cudaEvent_t e1 = pool_event(ctx);
    cudaEventRecord(e1, st);
    ctx->ev_phase.push_back({xs[0].kind, {pe0, e1}});
  }
  return WF_OK;
}

// Peer-memory phase whose receive side completes per source: copies and signals as in
// run_phase, then one wait per source followed by an event, so compute that needs only
// some sources can start before the rest have arrived (unit-pipelined R = 1 steps).
wf_status run_phase_per_source(wf_ctx* ctx, std::vector<Xfer>& xs, std::vector<wf_event>& trace, cudaStream_t st,
                               std::vector<cudaEvent_t>& src_ev) {
  const int me = ctx->rank;
  for (const Xfer& x : xs) {
    if (x.src == x.dst || !recorded(ctx, x.src)) continue;
    int64_t bytes = 0;
    for (const Seg& sg : x.segs) bytes += sg.bytes;
    trace.push_back(wf_event{x.pass, x.kind, x.step, x.src, x.dst, x.block, bytes});
  }
  WCK(dbg_check_segs(ctx, xs));
  if (ctx->debug & WF_DEBUG_NO_TRANSFER) return WF_OK;
  const int ch = st == ctx->comm_stream ? 1 : 0;
  cudaEvent_t pe0 = xs.empty() ? nullptr : prof_begin(ctx, st);
  for (const Xfer& x : xs) {
    if (x.src != me || x.pull || x.fused) continue;
    for (const Seg& sg : x.segs)
      if (sg.bytes && sg.src != sg.dst) CK(cudaMemcpyAsync(sg.dst, sg.src, sg.bytes, cudaMemcpyDefault, st));
  }
  SigArgs sig{}, none{};
  bool dst_done[kMaxRanks] = {}, src_done[kMaxRanks] = {};
  for (const Xfer& x : xs) {
    if (x.src == me && x.dst != me && !dst_done[x.dst]) {
      dst_done[x.dst] = true;
      sig.dst[sig.n] = flag_of(ctx, x.dst, ch * 64 + me);
      sig.val[sig.n++] = ++ctx->sent[ch][x.dst];
    }
  }
  WCK(sigwait(ctx, sig, none, st));
  for (const Xfer& x : xs) {
    if (x.dst == me && x.src != me && !src_done[x.src]) {
      src_done[x.src] = true;
      SigArgs w{};
      w.dst[0] = flag_of(ctx, me, ch * 64 + x.src);
      w.val[0] = ++ctx->rcvd[ch][x.src];
      w.n = 1;
      WCK(sigwait(ctx, none, w, st));
      CK(cudaEventRecord(src_ev[x.src], st));
    }
  }
  if (pe0) {
    cudaEvent_t e1 = pool_event(ctx);
    cudaEventRecord(e1, st);
    ctx->ev_phase.push_back({xs[0].kind, {pe0, e1}});
  }
  return WF_OK;
}

std::vector<cudaEvent_t>& source_events(wf_ctx* ctx, int n);

// pointer helpers that are null for non-local ranks
template <typename T>
T* at(T* base, int64_t off) {
  return base ? base + off : nullptr;
}

cudaEvent_t pool_event(wf_ctx* ctx) {
  cudaEvent_t e = nullptr;
  if (!ctx->ev_pool.empty()) {
    e = ctx->ev_pool.back();
    ctx->ev_pool.pop_back();
  } else {
    cudaEventCreate(&e);
  }
  return e;
}
cudaEvent_t prof_begin(wf_ctx* ctx, cudaStream_t st) {
  if (!ctx->profiling) return nullptr;
  cudaEvent_t e = pool_event(ctx);
  cudaEventRecord(e, st);
  return e;
}
void prof_end(wf_ctx* ctx, cudaStream_t st, cudaEvent_t e0,
              std::vector<std::pair<cudaEvent_t, cudaEvent_t>>& v) {
  if (!ctx->profiling || !e0) return;
  cudaEvent_t e1 = pool_event(ctx);
  cudaEventRecord(e1, st);
  v.push_back({e0, e1});
}

wf_status kcheck(wf_ctx* ctx, cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(ctx, WF_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
  ++ctx->launches;
  return WF_OK;
}

// ------------------------------------------------------------------ debug bounds checks
// A WF_DEBUG_CHECKS build (compute-sanitizer is not available on this pool) verifies that
// every copy segment, partial and accumulator pointer the schedule hands to a copy engine
// or a kernel lies inside one of the ranges the call may touch: the caller's tensors of
// this call, this rank's workspace, or a peer's mapped workspace.
void dbg_begin(wf_ctx* ctx, std::initializer_list<std::pair<const void*, size_t>> tensors) {
#ifdef WF_DEBUG_CHECKS
  ctx->dbg_ranges.clear();
  for (auto& t : tensors)
    if (t.first) ctx->dbg_ranges.push_back({static_cast<const char*>(t.first), t.second});
  if (ctx->ws) ctx->dbg_ranges.push_back({static_cast<const char*>(ctx->ws), ctx->ws_bytes});
  for (size_t r = 0; r < ctx->peer_base.size(); ++r)
    if (ctx->peer_base[r]) ctx->dbg_ranges.push_back({ctx->peer_base[r], ctx->ws_bytes});
#else
  (void)ctx;
  (void)tensors;
#endif
}
wf_status dbg_check(wf_ctx* ctx, const void* p, int64_t bytes, const char* what) {
#ifdef WF_DEBUG_CHECKS
  if (!p || bytes <= 0 || ctx->dry) return WF_OK;
  const char* c = static_cast<const char*>(p);
  for (auto& r : ctx->dbg_ranges)
    if (c >= r.first && c + bytes <= r.first + r.second) return WF_OK;
  char buf[160];
  std::snprintf(buf, sizeof(buf), "debug check: %s [%p, +%lld) outside every tensor / workspace of this call", what,
                p, static_cast<long long>(bytes));
  return fail(ctx, WF_ERR_ARG, buf);
#else
  (void)ctx;
  (void)p;
  (void)bytes;
  (void)what;
  return WF_OK;
#endif
}
// operands of one block-forward / block-backward launch
wf_status dbg_fwd(wf_ctx* ctx, const FwdArgs& a, const void* q, const void* k, const void* v, int64_t E) {
  WCK(dbg_check(ctx, q, a.nq * E * 2, "block-fwd Q"));
  WCK(dbg_check(ctx, k, a.nk * E * 2, "block-fwd K"));
  WCK(dbg_check(ctx, v, a.nk * E * 2, "block-fwd V"));
  WCK(dbg_check(ctx, a.o_in, a.nq * E * 4, "block-fwd O state in"));
  WCK(dbg_check(ctx, a.lse_in, static_cast<int64_t>(a.heads) * a.nq * 4, "block-fwd lse in"));
  WCK(dbg_check(ctx, a.o_out_f32, a.nq * E * 4, "block-fwd O state out"));
  WCK(dbg_check(ctx, a.o_out_bf16, a.nq * E * 2, "block-fwd O out"));
  return dbg_check(ctx, a.lse_out, static_cast<int64_t>(a.heads) * a.nq * 4, "block-fwd lse out");
}
wf_status dbg_bwd(wf_ctx* ctx, const BwdArgs& a, const void* q, const void* k, const void* v, const void* dO,
                  int64_t E) {
  WCK(dbg_check(ctx, q, a.nq * E * 2, "block-bwd Q"));
  WCK(dbg_check(ctx, dO, a.nq * E * 2, "block-bwd dO"));
  WCK(dbg_check(ctx, k, a.nk * E * 2, "block-bwd K"));
  WCK(dbg_check(ctx, v, a.nk * E * 2, "block-bwd V"));
  WCK(dbg_check(ctx, a.lse, static_cast<int64_t>(a.heads) * a.nq * 4, "block-bwd LSE"));
  WCK(dbg_check(ctx, a.dsum, static_cast<int64_t>(a.heads) * a.nq * 4, "block-bwd D"));
  WCK(dbg_check(ctx, a.dq_acc, a.nq * E * 4, "block-bwd dQ accumulator"));
  WCK(dbg_check(ctx, a.dk_acc, a.nk * E * 4, "block-bwd dK accumulator"));
  WCK(dbg_check(ctx, a.dv_acc, a.nk * E * 4, "block-bwd dV accumulator"));
  WCK(dbg_check(ctx, a.dk_out, a.nk * E * 2, "block-bwd dK out"));
  return dbg_check(ctx, a.dv_out, a.nk * E * 2, "block-bwd dV out");
}
wf_status dbg_check_segs(wf_ctx* ctx, const std::vector<Xfer>& xs) {
#ifdef WF_DEBUG_CHECKS
  for (const Xfer& x : xs)
    for (const Seg& sg : x.segs) {
      if (!local(ctx, x.src) && !ctx->ipc) continue;
      WCK(dbg_check(ctx, sg.src, sg.bytes, "segment source"));
      WCK(dbg_check(ctx, sg.dst, sg.bytes, "segment destination"));
    }
#else
  (void)ctx;
  (void)xs;
#endif
  return WF_OK;
}

// ------------------------------------------------------------------ peer-memory sync helpers
// Per-call barrier of all ranks: no peer writes into my workspace before I have finished
// reading what the previous call left there (stream order puts this after my previous work).
wf_status ipc_barrier(wf_ctx* ctx, cudaStream_t st) {
  if (!ctx->ipc || ctx->dry || (ctx->debug & WF_DEBUG_NO_TRANSFER)) return WF_OK;
  const int P = ctx->plan.P, me = ctx->rank;
  ++ctx->epoch;
  SigArgs sig{}, wt{};
  for (int r = 0; r < P; ++r) {
    if (r == me) continue;
    sig.dst[sig.n] = flag_of(ctx, r, 192 + me);
    sig.val[sig.n++] = ctx->epoch;
    wt.dst[wt.n] = flag_of(ctx, me, 192 + r);
    wt.val[wt.n++] = ctx->epoch;
  }
  WCK(sigwait(ctx, sig, wt, st));
  return WF_OK;
}
// Tell `to` that I finished reading the ring slot it fills (one more released slot).
wf_status ipc_ack(wf_ctx* ctx, int to, cudaStream_t st) {
  if (!ctx->ipc || ctx->dry || (ctx->debug & WF_DEBUG_NO_TRANSFER) || to == ctx->rank) return WF_OK;
  SigArgs sig{}, wt{};
  sig.dst[0] = flag_of(ctx, to, 128 + ctx->rank);
  sig.val[0] = ++ctx->acks_sent[to];
  sig.n = 1;
  WCK(sigwait(ctx, sig, wt, st));
  return WF_OK;
}
// Wait until `from` has released `count` slots in this ring loop (ack_base counts the
// releases of earlier loops; every loop releases R - 1 slots).
wf_status ipc_wait_ack(wf_ctx* ctx, int from, uint32_t count, cudaStream_t st) {
  if (!ctx->ipc || ctx->dry || (ctx->debug & WF_DEBUG_NO_TRANSFER) || from == ctx->rank || count == 0) return WF_OK;
  SigArgs sig{}, wt{};
  wt.dst[0] = flag_of(ctx, ctx->rank, 128 + from);
  wt.val[0] = ctx->ack_base[from] + count;
  wt.n = 1;
  WCK(sigwait(ctx, sig, wt, st));
  return WF_OK;
}
std::vector<cudaEvent_t>& source_events(wf_ctx* ctx, int n) {
  while (static_cast<int>(ctx->ev_src.size()) < n) {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ctx->ev_src.push_back(e);
  }
  return ctx->ev_src;
}
cudaEvent_t step_event(wf_ctx* ctx, int i) {
  while (static_cast<int>(ctx->ev_step.size()) <= i) {
    cudaEvent_t e = nullptr;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    ctx->ev_step.push_back(e);
  }
  return ctx->ev_step[i];
}
// join the comm stream back into the caller's stream
wf_status join_comm(wf_ctx* ctx, cudaStream_t st) {
  if (ctx->dry || ctx->emulated) return WF_OK;
  CK(cudaEventRecord(ctx->ev_c, ctx->comm_stream));
  CK(cudaStreamWaitEvent(st, ctx->ev_c, 0));
  return WF_OK;
}

// Unit-pipelined passes run the query units of member a in the order a, a+1, ..., a+C-1
// (team-relative): member i's last unit is that of member i-1.
bool last_unit_of(int C, int i, int j) { return (j + 1) % C == i; }

// push a finished partial into its owner's slot: a copy-engine copy on the comm stream after
// the producing kernel (peer memory), or a device copy in stream order (emulated)
wf_status push_segs(wf_ctx* ctx, const Seg* segs, int nseg, cudaStream_t st) {
  for (int i = 0; i < nseg; ++i) {
    WCK(dbg_check(ctx, segs[i].src, segs[i].bytes, "pushed partial source"));
    WCK(dbg_check(ctx, segs[i].dst, segs[i].bytes, "pushed partial destination"));
  }
  if (ctx->ipc) {
    CK(cudaEventRecord(ctx->ev_b, st));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_b, 0));
  }
  for (int i = 0; i < nseg; ++i)
    CK(cudaMemcpyAsync(segs[i].dst, segs[i].src, segs[i].bytes, cudaMemcpyDefault, ctx->ipc ? ctx->comm_stream : st));
  return WF_OK;
}

// a reduce-scatter phase whose senders pushed part of it from the comm stream: the signals
// go out from the comm stream after those pushes and after my compute, the caller's stream
// waits for the matching arrivals
wf_status run_phase_after_pushes(wf_ctx* ctx, std::vector<Xfer>& xs, std::vector<wf_event>& tr, cudaStream_t st,
                                 bool pushed) {
  if (!pushed || !ctx->ipc) return run_phase(ctx, xs, tr, st);
  CK(cudaEventRecord(ctx->ev_b, st));
  CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_b, 0));
  WCK(run_phase(ctx, xs, tr, ctx->comm_stream));
  CK(cudaEventRecord(ctx->ev_c, ctx->comm_stream));
  CK(cudaStreamWaitEvent(st, ctx->ev_c, 0));
  return WF_OK;
}

// ------------------------------------------------------------------ forward
wf_status forward(wf_ctx* ctx, const Geo& g, const bf16* Q, const bf16* K, const bf16* V, bf16* O, float* LSE,
                  cudaStream_t st) {
  const Plan& pl = ctx->plan;
  const int P = g.P, C = g.C, R = g.R;
  const int64_t n = g.n, E = g.E, h = g.h;
  auto Qin = [&](int r) { return local(ctx, r) ? Q + (ctx->emulated ? r * n * E : 0) : nullptr; };
  auto Kin = [&](int r) { return local(ctx, r) ? K + (ctx->emulated ? r * n * E : 0) : nullptr; };
  auto Vin = [&](int r) { return local(ctx, r) ? V + (ctx->emulated ? r * n * E : 0) : nullptr; };
  auto Oout = [&](int r) { return local(ctx, r) ? O + (ctx->emulated ? r * n * E : 0) : nullptr; };
  auto Lout = [&](int r) { return local(ctx, r) ? LSE + (ctx->emulated ? r * n * h : 0) : nullptr; };
  auto lp = [&](int r, auto* p) { return addressable(ctx, r) ? p : decltype(p)(nullptr); };
  auto& tr = ctx->trace_fwd;
  tr.clear();
  {
    const int64_t nr = ctx->emulated ? P : 1;
    dbg_begin(ctx, {{Q, nr * n * E * 2}, {K, nr * n * E * 2}, {V, nr * n * E * 2}, {O, nr * n * E * 2},
                    {LSE, nr * n * h * 4}});
  }
  // gathers already delivered by wf_qkv_proj's epilogue (same tensors, same geometry)
  const int64_t key[4] = {g.N, g.h, g.d, g.causal};
  const bool pre = ctx->proj_q && ctx->proj_seq + 1 == ctx->seq && ctx->proj_q == Q && ctx->proj_k == K &&
                   ctx->proj_v == V && std::equal(key, key + 4, ctx->proj_key);
  ctx->proj_q = ctx->proj_k = ctx->proj_v = nullptr;
  WCK(ipc_barrier(ctx, st));

  // Team tensors (C = 1: the caller's shard itself).
  auto qteam = [&](int r) -> const bf16* { return C > 1 ? lp(r, B(ctx, r).qt) : Qin(r); };
  auto kteam = [&](int r) -> const bf16* { return C > 1 ? lp(r, B(ctx, r).kt) : Kin(r); };
  auto vteam = [&](int r) -> const bf16* { return C > 1 ? lp(r, B(ctx, r).vt) : Vin(r); };

  // Extension regime over peer memory (R = 1): unit-pipelined.  The team gather of Q and
  // the K/V slice pull run on the comm stream with one completion event per source rank;
  // the step is cut into (query unit, key unit) launches that merge into the same (O, lse)
  // state, the locally present units first, so the transfers overlap the compute.
  // The K/V units rank r attends first: its slice (extension) or its initial team block
  // team(recv[r]) (paper regime; pulled unit by unit in the DIRECT-PULL variant).
  auto kfirst = [&](int r) { return g.paper ? (pl.recv[r] / C) * C : (r % C) * g.W; };
  const int kcount = g.paper ? C : g.W;
  const bool unitpipe = (ctx->ipc || ctx->emulated) && C > 1 && !g.paper;
  if (unitpipe) {
    std::vector<cudaEvent_t>& sev = source_events(ctx, P);
    CK(cudaEventRecord(ctx->ev_a, st));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0));
    std::vector<Xfer> xs;
    for (int r = 0; r < P; ++r) {
      const int tr_ = r / C, j = r - tr_ * C;
      for (int p = tr_ * C; p < tr_ * C + C; ++p) {
        if (p == r) continue;  // my own rows are read from the caller's buffer
        Xfer x{0, WF_KIND_AG_Q, -1, r, p, r, {}};
        x.segs.push_back({Qin(r), at(lp(p, B(ctx, p).qt), j * n * E), n * E * 2});
        x.fused = pre;
        xs.push_back(x);
      }
      for (int u = kfirst(r); u < kfirst(r) + kcount; ++u) {
        if (u == r) continue;
        const int64_t off = static_cast<int64_t>(u - kfirst(r)) * n * E;
        Xfer x{0, WF_KIND_SLICE_KV, -1, u, r, u, {}};
        x.fused = pre;
        x.segs.push_back({Kin(u), at(lp(r, B(ctx, r).rk[0]), off), n * E * 2});
        x.segs.push_back({Vin(u), at(lp(r, B(ctx, r).rv[0]), off), n * E * 2});
        xs.push_back(x);
      }
    }
    if (ctx->ipc)
      WCK(run_phase_per_source(ctx, xs, tr, ctx->comm_stream, sev));
    else
      WCK(run_phase(ctx, xs, tr, st));  // emulated: device copies in stream order
    for (int me = 0; me < P; ++me) {
    if (!local(ctx, me)) continue;
    const int t = me / C, a = me % C;
    RankBufs& b = B(ctx, me);
    std::vector<int> qorder, korder;
    for (int i = 0; i < C; ++i) qorder.push_back(t * C + (a + i) % C);  // own unit first
    for (int i = 0; i < kcount; ++i) {
      const int u = kfirst(me) + i;
      if (u == me) korder.insert(korder.begin(), u); else korder.push_back(u);
    }
    for (size_t qi = 0; qi < qorder.size(); ++qi) {
      const int qj = qorder[qi];
      const int jm = qj - t * C;
      const bf16* qp = qj == me ? Qin(me) : b.qt + jm * n * E;
      for (size_t ki = 0; ki < korder.size(); ++ki) {
        const int u = korder[ki];
        const int64_t koff = static_cast<int64_t>(u - kfirst(me)) * n * E;
        const bf16* kp = u == me ? Kin(me) : b.rk[0] + koff;
        const bf16* vp = u == me ? Vin(me) : b.rv[0] + koff;
        if (ctx->ipc && qj != me) CK(cudaStreamWaitEvent(st, sev[qj], 0));
        if (ctx->ipc && u != me) CK(cudaStreamWaitEvent(st, sev[u], 0));
        FwdArgs fa{};
        fa.nq = g.n;
        fa.nk = g.n;
        fa.heads = g.h;
        fa.causal = g.causal;
        fa.qpos = units_table(g, qj, 1);
        fa.kpos = units_table(g, u, 1);
        fa.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(g.d));
        fa.o_in = ki > 0 ? b.o_state + jm * n * E : nullptr;
        fa.lse_in = ki > 0 ? b.lse_state + jm * h * n : nullptr;
        fa.o_out_f32 = b.o_state + jm * n * E;
        fa.lse_out = b.lse_state + jm * h * n;
        fa.lse_blk = g.n;
        CUtensorMap tq, tk, tv;
        if (!make_tmap_rows(&tq, qp, fa.nq, g.h, g.d) || !make_tmap_rows(&tk, kp, fa.nk, g.h, g.d) ||
            !make_tmap_rows(&tv, vp, fa.nk, g.h, g.d))
          return fail(ctx, WF_ERR_ARG, "TMA map encode failed (alignment?)");
        WCK(dbg_fwd(ctx, fa, qp, kp, vp, E));
        cudaEvent_t e0 = prof_begin(ctx, st);
        WCK(kcheck(ctx, launch_block_fwd(tq, tk, tv, fa, g.d, st), "block_fwd"));
        prof_end(ctx, st, e0, ctx->ev_fwd);
      }
      // member qj's partial is final; unless it is my last unit (which its owner reads in
      // place), push it into qj's merge slot while the next units run
      if (qj != me && qi + 1 < qorder.size() && !(ctx->debug & WF_DEBUG_NO_TRANSFER)) {
        const Seg segs[2] = {{b.o_state + jm * n * E, B(ctx, qj).rs_o + a * n * E, n * E * 4},
                             {b.lse_state + jm * h * n, B(ctx, qj).rs_lse + a * h * n, h * n * 4}};
        WCK(push_segs(ctx, segs, 2, st));
      }
    }
    }  // ranks
  } else {
    // Alg. 1 l.1: team all-gather (member-major).
    if (C > 1) {
      std::vector<Xfer> xs;
      for (int r = 0; r < P; ++r) {
        const int t = r / C, j = r - t * C;
        for (int p = t * C; p < t * C + C; ++p) {
          Xfer x{0, WF_KIND_AG_Q, -1, r, p, r, {}};
          x.segs.push_back({Qin(r), at(lp(p, B(ctx, p).qt), j * n * E), n * E * 2});
          x.fused = pre;
          xs.push_back(x);
          if (g.paper && !g.direct) {
            Xfer y{0, WF_KIND_AG_KV, -1, r, p, r, {}};
            y.fused = pre;
            y.segs.push_back({Kin(r), at(lp(p, B(ctx, p).kt), j * n * E), n * E * 2});
            y.segs.push_back({Vin(r), at(lp(p, B(ctx, p).vt), j * n * E), n * E * 2});
            xs.push_back(y);
          }
        }
      }
      WCK(run_phase(ctx, xs, tr, st));
    }

    // Per rank: pointers of the K/V block in ring slot 0/1.
    std::vector<const bf16*> ck0(P, nullptr), cv0(P, nullptr);
    if (g.paper && !g.direct) {
      // Alg. 1 l.2: initial shuffle to init_send (a self "send" keeps the block in place).
      std::vector<Xfer> xs;
      for (int r = 0; r < P; ++r) {
        const int dst = pl.send[r];
        if (dst == r) continue;
        Xfer x{0, WF_KIND_INIT_KV, -1, r, dst, r / C, {}};
        x.segs.push_back({kteam(r), lp(dst, B(ctx, dst).rk[0]), static_cast<int64_t>(C) * n * E * 2});
        x.segs.push_back({vteam(r), lp(dst, B(ctx, dst).rv[0]), static_cast<int64_t>(C) * n * E * 2});
        xs.push_back(x);
      }
      WCK(run_phase(ctx, xs, tr, st));
      for (int r = 0; r < P; ++r) {
        if (pl.send[r] == r) {  // recv[r] == r too
          ck0[r] = kteam(r);
          cv0[r] = vteam(r);
        } else {
          ck0[r] = lp(r, B(ctx, r).rk[0]);
          cv0[r] = lp(r, B(ctx, r).rv[0]);
        }
      }
    } else {
      // extension: member a pulls K/V slice a straight from the unit owners (and, in the
      // DIRECT-PULL variant, every rank its initial team block)
      std::vector<Xfer> xs;
      for (int r = 0; r < P; ++r) {
        for (int u = kfirst(r); u < kfirst(r) + kcount; ++u) {
          const int64_t off = static_cast<int64_t>(u - kfirst(r)) * n * E;
          Xfer x{0, WF_KIND_SLICE_KV, -1, u, r, u, {}};
          x.fused = pre;
          x.segs.push_back({Kin(u), at(lp(r, B(ctx, r).rk[0]), off), n * E * 2});
          x.segs.push_back({Vin(u), at(lp(r, B(ctx, r).rv[0]), off), n * E * 2});
          xs.push_back(x);
        }
      }
      WCK(run_phase(ctx, xs, tr, st));
      for (int r = 0; r < P; ++r) {
        ck0[r] = lp(r, B(ctx, r).rk[0]);
        cv0[r] = lp(r, B(ctx, r).rv[0]);
      }
    }

    // Alg. 1 l.5-10: R ring steps, K/V double buffered; the transfer of block s+1
    // (comm stream) is posted before the block kernel of step s.
    const bool overlap = !ctx->emulated && !ctx->dry && R > 1;
    auto slot_k = [&](int r, int s) -> const bf16* { return s == 0 ? ck0[r] : lp(r, B(ctx, r).rk[s & 1]); };
    auto slot_v = [&](int r, int s) -> const bf16* { return s == 0 ? cv0[r] : lp(r, B(ctx, r).rv[s & 1]); };
    auto compute = [&](int r, int s) -> wf_status {
      RankBufs& b = B(ctx, r);
      FwdArgs a{};
      a.nq = C * g.n;
      a.nk = g.Bk;
      a.heads = g.h;
      a.causal = g.causal;
      a.qpos = units_table(g, (r / C) * C, C);
      a.kpos = g.paper ? units_table(g, pl.block_at(r, s) * C, C) : units_table(g, (r % C) * g.W, g.W);
      a.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(g.d));
      a.o_in = s > 0 ? b.o_state : nullptr;
      a.lse_in = s > 0 ? b.lse_state : nullptr;
      a.lse_blk = g.n;
      if (s < R - 1) {  // intermediate step: fp32 (O, lse) state, merged in place next step
        a.o_out_f32 = b.o_state;
        a.lse_out = b.lse_state;
      } else if (C == 1) {  // final output
        a.o_out_bf16 = Oout(r);
        a.lse_out = Lout(r);
      } else {  // this member's fp32 partial for the team rows (reading c17)
        a.o_out_f32 = b.o_state;
        a.lse_out = b.lse_state;
      }
      if (ctx->dry) return WF_OK;
      CUtensorMap tq, tk, tv;
      if (!make_tmap_rows(&tq, qteam(r), a.nq, g.h, g.d) || !make_tmap_rows(&tk, slot_k(r, s), a.nk, g.h, g.d) ||
          !make_tmap_rows(&tv, slot_v(r, s), a.nk, g.h, g.d))
        return fail(ctx, WF_ERR_ARG, "TMA map encode failed (alignment?)");
      WCK(dbg_fwd(ctx, a, qteam(r), slot_k(r, s), slot_v(r, s), E));
      cudaEvent_t e0 = prof_begin(ctx, st);
      wf_status ks = kcheck(ctx, launch_block_fwd(tq, tk, tv, a, g.d, st), "block_fwd");
      prof_end(ctx, st, e0, ctx->ev_fwd);
      return ks;
    };
    if (overlap) CK(cudaEventRecord(ctx->ev_a, st));  // slot 0 ready
    for (int s = 0; s < R; ++s) {
      std::vector<Xfer> xs;
      if (s < R - 1) {
        for (int r = 0; r < P; ++r) {
          const int dst = pl.next[r];
          Xfer x{0, WF_KIND_RING_KV, s, r, dst, g.paper ? pl.block_at(r, s) : r, {}};
          x.segs.push_back({slot_k(r, s), lp(dst, B(ctx, dst).rk[(s + 1) & 1]), static_cast<int64_t>(g.Bk) * E * 2});
          x.segs.push_back({slot_v(r, s), lp(dst, B(ctx, dst).rv[(s + 1) & 1]), static_cast<int64_t>(g.Bk) * E * 2});
          xs.push_back(x);
        }
        if (overlap) {
          // Alg. 1 l.8 with peer copies: the comm stream pushes block s into next's other
          // slot as soon as next has released it (its step s-1), independent of my compute.
          if (s == 0) CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0));
          WCK(ipc_wait_ack(ctx, pl.next[ctx->rank], static_cast<uint32_t>(s), ctx->comm_stream));
          WCK(run_phase(ctx, xs, tr, ctx->comm_stream, kPhaseSend));
        }
      }
      for (int r = 0; r < P; ++r)
        if (local(ctx, r)) WCK(compute(r, s));
      if (s < R - 1) {
        if (overlap) {
          // my slot s is free again once my kernel has read it AND my comm stream has
          // forwarded it to next (the send above): release it from the comm stream after
          // both, then wait for block s+1 from last
          CK(cudaEventRecord(ctx->ev_b, st));
          CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_b, 0));
          WCK(ipc_ack(ctx, pl.last[ctx->rank], ctx->comm_stream));
          WCK(run_phase(ctx, xs, tr, ctx->comm_stream, kPhaseWait));
          CK(cudaEventRecord(step_event(ctx, s), ctx->comm_stream));
          CK(cudaStreamWaitEvent(st, step_event(ctx, s), 0));
        } else {
          WCK(run_phase(ctx, xs, tr, st));
        }
      }
    }
    if (overlap && !(ctx->debug & WF_DEBUG_NO_TRANSFER)) ctx->ack_base[pl.next[ctx->rank]] += R - 1;

  }

  // Alg. 1 l.11: ReduceScatter_combine -- partial rows to their owner, LSE-merge there.
  const bool nt = (ctx->debug & WF_DEBUG_NO_TRANSFER) != 0;
  if (C > 1) {
    std::vector<Xfer> xs;
    for (int r = 0; r < P; ++r) {
      const int t = r / C, j = r - t * C;
      for (int p = t * C; p < t * C + C; ++p) {
        if (p == r) continue;
        const int jp = p - t * C;
        // peer-memory transport: the owner's merge kernel reads the partial in place
        // (fused reduce-scatter); otherwise it is copied into the owner's slot first.
        // Unit-pipelined: all but the sender's last unit were pushed already (above).
        const bool pushed = unitpipe && !last_unit_of(C, j, jp);
        Xfer x{0, WF_KIND_RS_O, R, r, p, p, {}, ctx->ipc && !pushed, pushed};
        x.segs.push_back({at(lp(r, B(ctx, r).o_state), jp * n * E), at(lp(p, B(ctx, p).rs_o), j * n * E), n * E * 4});
        xs.push_back(x);
        Xfer y{0, WF_KIND_RS_LSE, R, r, p, p, {}, ctx->ipc && !pushed, pushed};
        y.segs.push_back({at(lp(r, B(ctx, r).lse_state), jp * h * n), at(lp(p, B(ctx, p).rs_lse), j * h * n), h * n * 4});
        xs.push_back(y);
      }
    }
    WCK(run_phase_after_pushes(ctx, xs, tr, st, unitpipe));
    for (int r = 0; r < P; ++r) {
      if (!local(ctx, r)) continue;
      RankBufs& b = B(ctx, r);
      const int j = r % C;
      MergeArgs m{};
      m.rows = g.n;
      m.heads = g.h;
      m.D = g.d;
      m.nparts = C;
      const int t0 = (r / C) * C;
      for (int i = 0; i < C; ++i) {
        if (i == j || nt) {  // own partial (nt: no-transfer timing baseline, local reads only)
          m.o[i] = b.o_state + i * n * E;
          m.lse[i] = b.lse_state + i * h * n;
        } else if (ctx->ipc && (!unitpipe || last_unit_of(C, i, j))) {  // read in place over NVLink
          m.o[i] = B(ctx, t0 + i).o_state + j * n * E;
          m.lse[i] = B(ctx, t0 + i).lse_state + j * h * n;
        } else {
          m.o[i] = b.rs_o + i * n * E;
          m.lse[i] = b.rs_lse + i * h * n;
        }
        m.lse_stride[i] = n;
      }
      m.out = Oout(r);
      m.lse_out = Lout(r);
      for (int i = 0; i < C; ++i) {
        WCK(dbg_check(ctx, m.o[i], n * E * 4, "merge partial"));
        WCK(dbg_check(ctx, m.lse[i], h * n * 4, "merge lse partial"));
      }
      if (!ctx->dry) WCK(kcheck(ctx, launch_merge(m, st), "merge"));
    }
  }
  return join_comm(ctx, st);
}

// ------------------------------------------------------------------ backward
wf_status backward(wf_ctx* ctx, const Geo& g, const bf16* dO, const bf16* Q, const bf16* K, const bf16* V,
                   const bf16* O, const float* LSE, bf16* dQ, bf16* dK, bf16* dV, cudaStream_t st) {
  const Plan& pl = ctx->plan;
  const int P = g.P, C = g.C, R = g.R;
  const int64_t n = g.n, E = g.E, h = g.h, team = static_cast<int64_t>(C) * n * E;
  auto off = [&](int r, int64_t per) { return ctx->emulated ? r * per : 0; };
  auto L = [&](int r, auto* p, int64_t per) { return local(ctx, r) ? p + off(r, per) : decltype(p)(nullptr); };
  auto lp = [&](int r, auto* p) { return addressable(ctx, r) ? p : decltype(p)(nullptr); };
  auto& tr = ctx->trace_bwd;
  tr.clear();
  {
    const int64_t nr = ctx->emulated ? P : 1;
    dbg_begin(ctx, {{dO, nr * n * E * 2}, {Q, nr * n * E * 2}, {K, nr * n * E * 2}, {V, nr * n * E * 2},
                    {O, nr * n * E * 2}, {LSE, nr * n * h * 4}, {dQ, nr * n * E * 2}, {dK, nr * n * E * 2},
                    {dV, nr * n * E * 2}});
  }
  const bool nt = (ctx->debug & WF_DEBUG_NO_TRANSFER) != 0;
  WCK(ipc_barrier(ctx, st));

  // D = rowsum(dO o O) on own rows (reading c12), stored with this rank's LSE in the form
  // the block backward consumes (-D / sqrt(d), -LSE log2(e)); these are what the team
  // gathers and the Q-package carry (same bytes as the raw statistics).
  for (int r = 0; r < P; ++r) {
    if (!local(ctx, r) || ctx->dry) continue;
    WCK(kcheck(ctx,
               launch_dsum(L(r, dO, n * E), L(r, O, n * E), L(r, LSE, n * h), B(ctx, r).dsum, B(ctx, r).nlse, g.n,
                           g.h, g.d, 1.f / std::sqrt(static_cast<float>(g.d)), st),
               "dsum"));
  }
  auto qteam = [&](int r) -> const bf16* { return C > 1 ? lp(r, B(ctx, r).qt) : L(r, Q, n * E); };
  auto doteam = [&](int r) -> const bf16* { return C > 1 ? lp(r, B(ctx, r).t_do) : L(r, dO, n * E); };
  auto lseteam = [&](int r) -> const float* { return C > 1 ? lp(r, B(ctx, r).t_lse) : lp(r, B(ctx, r).nlse); };
  auto dsteam = [&](int r) -> const float* { return C > 1 ? lp(r, B(ctx, r).t_dsum) : lp(r, B(ctx, r).dsum); };
  auto kteam = [&](int r) -> const bf16* { return C > 1 ? lp(r, B(ctx, r).kt) : L(r, K, n * E); };
  auto vteam = [&](int r) -> const bf16* { return C > 1 ? lp(r, B(ctx, r).vt) : L(r, V, n * E); };

  // package slots: step 0 = own team (aliases); later steps in the receive buffers
  auto pq = [&](int r, int s) -> const bf16* { return s == 0 ? qteam(r) : lp(r, B(ctx, r).pq[s & 1]); };
  auto pdo = [&](int r, int s) -> const bf16* { return s == 0 ? doteam(r) : lp(r, B(ctx, r).pdo[s & 1]); };
  auto plse = [&](int r, int s) -> const float* { return s == 0 ? lseteam(r) : lp(r, B(ctx, r).plse[s & 1]); };
  auto pds = [&](int r, int s) -> const float* { return s == 0 ? dsteam(r) : lp(r, B(ctx, r).pdsum[s & 1]); };
  auto pdq = [&](int r, int s) -> float* { return lp(r, B(ctx, r).pdq[s & 1]); };
  std::vector<int> pkg_team(P);
  for (int r = 0; r < P; ++r) pkg_team[r] = r / C;
  auto kfirst = [&](int r) { return g.paper ? (pl.recv[r] / C) * C : (r % C) * g.W; };
  const int kcount = g.paper ? C : g.W;
  const bool unitpipe = (ctx->ipc || ctx->emulated) && C > 1 && !g.paper;
  if (unitpipe) {
    // Extension regime over peer memory (R = 1): unit-pipelined like the forward.  The
    // gathers of Q, dO, LSE, D and the K/V slice pull run on the comm stream with one
    // completion event per source rank; the step is cut into (query unit, key unit)
    // launches, locally present units first.  dQ rows accumulate per query unit, dK/dV
    // rows per key unit.  (Emulated mode runs the same decomposition for every virtual
    // rank, so it is tested at every (P, C) on one GPU.)
    std::vector<cudaEvent_t>& sev = source_events(ctx, P);
    CK(cudaEventRecord(ctx->ev_a, st));  // after D of my rows
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0));
    std::vector<Xfer> xs;
    for (int r = 0; r < P; ++r) {
      const int tr_ = r / C, j = r - tr_ * C;
      for (int p = tr_ * C; p < tr_ * C + C; ++p) {
        if (p == r) continue;
        Xfer x{1, WF_KIND_AG_QDO, -1, r, p, r, {}};
        x.segs.push_back({L(r, Q, n * E), at(lp(p, B(ctx, p).qt), j * n * E), n * E * 2});
        x.segs.push_back({L(r, dO, n * E), at(lp(p, B(ctx, p).t_do), j * n * E), n * E * 2});
        xs.push_back(x);
        Xfer y{1, WF_KIND_AG_STATS, -1, r, p, r, {}};
        y.segs.push_back({lp(r, B(ctx, r).nlse), at(lp(p, B(ctx, p).t_lse), j * h * n), h * n * 4});
        y.segs.push_back({lp(r, B(ctx, r).dsum), at(lp(p, B(ctx, p).t_dsum), j * h * n), h * n * 4});
        xs.push_back(y);
      }
      for (int u = kfirst(r); u < kfirst(r) + kcount; ++u) {
        if (u == r) continue;
        const int64_t o = static_cast<int64_t>(u - kfirst(r)) * n * E;
        Xfer x{1, WF_KIND_SLICE_KV, -1, u, r, u, {}};
        x.segs.push_back({L(u, K, n * E), at(lp(r, B(ctx, r).rk[0]), o), n * E * 2});
        x.segs.push_back({L(u, V, n * E), at(lp(r, B(ctx, r).rv[0]), o), n * E * 2});
        xs.push_back(x);
      }
    }
    if (ctx->ipc)
      WCK(run_phase_per_source(ctx, xs, tr, ctx->comm_stream, sev));
    else
      WCK(run_phase(ctx, xs, tr, st));
    for (int me = 0; me < P; ++me) {
    if (!local(ctx, me)) continue;
    const int t = me / C, a = me % C;
    RankBufs& b = B(ctx, me);
    CK(cudaMemsetAsync(b.pdq[0], 0, team * 4, st));
    std::vector<int> qorder, korder;
    for (int i = 0; i < C; ++i) qorder.push_back(t * C + (a + i) % C);
    for (int i = 0; i < kcount; ++i) {
      const int u = kfirst(me) + i;
      if (u == me) korder.insert(korder.begin(), u); else korder.push_back(u);
    }
    for (size_t qi = 0; qi < qorder.size(); ++qi) {
      const int qj = qorder[qi];
      const int jm = qj - t * C;
      const bool own = qj == me;
      const bf16* qp = own ? L(me, Q, n * E) : b.qt + jm * n * E;
      const bf16* dop = own ? L(me, dO, n * E) : b.t_do + jm * n * E;
      for (size_t ki = 0; ki < korder.size(); ++ki) {
        const int u = korder[ki];
        const int64_t koff = static_cast<int64_t>(u - kfirst(me)) * n * E;
        const bf16* kp = u == me ? L(me, K, n * E) : b.rk[0] + koff;
        const bf16* vp = u == me ? L(me, V, n * E) : b.rv[0] + koff;
        if (ctx->ipc && !own) CK(cudaStreamWaitEvent(st, sev[qj], 0));
        if (ctx->ipc && u != me) CK(cudaStreamWaitEvent(st, sev[u], 0));
        BwdArgs ba{};
        ba.nq = g.n;
        ba.nk = g.n;
        ba.heads = g.h;
        ba.causal = g.causal;
        ba.qpos = units_table(g, qj, 1);
        ba.kpos = units_table(g, u, 1);
        ba.scale = 1.f / std::sqrt(static_cast<float>(g.d));
        ba.scale_log2 = 1.4426950408889634f * ba.scale;
        ba.lse = own ? b.nlse : b.t_lse + jm * h * n;
        ba.dsum = own ? b.dsum : b.t_dsum + jm * h * n;
        ba.stat_blk = g.n;
        ba.dq_acc = b.pdq[0] + jm * n * E;
        ba.dk_acc = b.dk_acc + koff;
        ba.dv_acc = b.dv_acc + koff;
        ba.dkv_accumulate = qi > 0;
        CUtensorMap tq, tk, tv, tdo;
        if (!make_tmap_rows(&tq, qp, ba.nq, g.h, g.d) || !make_tmap_rows(&tk, kp, ba.nk, g.h, g.d) ||
            !make_tmap_rows(&tv, vp, ba.nk, g.h, g.d) || !make_tmap_rows(&tdo, dop, ba.nq, g.h, g.d))
          return fail(ctx, WF_ERR_ARG, "TMA map encode failed (alignment?)");
        WCK(dbg_bwd(ctx, ba, qp, kp, vp, dop, E));
        cudaEvent_t e0 = prof_begin(ctx, st);
        WCK(kcheck(ctx, launch_block_bwd(tq, tk, tv, tdo, ba, g.d, st), "block_bwd"));
        prof_end(ctx, st, e0, ctx->ev_bwd);
      }
      // member qj's dQ partial is final: pushed like the forward partials
      if (!own && qi + 1 < qorder.size() && !(ctx->debug & WF_DEBUG_NO_TRANSFER)) {
        const Seg sg{b.pdq[0] + jm * n * E, B(ctx, qj).rsq + a * n * E, n * E * 4};
        WCK(push_segs(ctx, &sg, 1, st));
      }
    }
    }  // ranks
  } else {
    // team gathers: Q + dO, LSE + D, and (paper regime) K + V
    if (C > 1) {
      std::vector<Xfer> xs;
      for (int r = 0; r < P; ++r) {
        const int t = r / C, j = r - t * C;
        for (int p = t * C; p < t * C + C; ++p) {
          Xfer x{1, WF_KIND_AG_QDO, -1, r, p, r, {}};
          x.segs.push_back({L(r, Q, n * E), at(lp(p, B(ctx, p).qt), j * n * E), n * E * 2});
          x.segs.push_back({L(r, dO, n * E), at(lp(p, B(ctx, p).t_do), j * n * E), n * E * 2});
          xs.push_back(x);
          Xfer y{1, WF_KIND_AG_STATS, -1, r, p, r, {}};
          y.segs.push_back({lp(r, B(ctx, r).nlse), at(lp(p, B(ctx, p).t_lse), j * h * n), h * n * 4});
          y.segs.push_back({lp(r, B(ctx, r).dsum), at(lp(p, B(ctx, p).t_dsum), j * h * n), h * n * 4});
          xs.push_back(y);
          if (g.paper && !g.direct) {
            Xfer z{1, WF_KIND_AG_KV, -1, r, p, r, {}};
            z.segs.push_back({L(r, K, n * E), at(lp(p, B(ctx, p).kt), j * n * E), n * E * 2});
            z.segs.push_back({L(r, V, n * E), at(lp(p, B(ctx, p).vt), j * n * E), n * E * 2});
            xs.push_back(z);
          }
        }
      }
      WCK(run_phase(ctx, xs, tr, st));
    }

    // stationary K/V block: the init-shuffle block (paper) or the slice (extension)
    std::vector<const bf16*> sk(P, nullptr), sv(P, nullptr);
    {
      std::vector<Xfer> xs;
      for (int r = 0; r < P; ++r) {
        if (g.paper && !g.direct) {
          const int dst = pl.send[r];
          if (dst == r) continue;
          Xfer x{1, WF_KIND_INIT_KV, -1, r, dst, r / C, {}};
          x.segs.push_back({kteam(r), lp(dst, B(ctx, dst).rk[0]), team * 2});
          x.segs.push_back({vteam(r), lp(dst, B(ctx, dst).rv[0]), team * 2});
          xs.push_back(x);
        } else {
          for (int u = kfirst(r); u < kfirst(r) + kcount; ++u) {
            const int64_t o = static_cast<int64_t>(u - kfirst(r)) * n * E;
            Xfer x{1, WF_KIND_SLICE_KV, -1, u, r, u, {}};
            x.segs.push_back({L(u, K, n * E), at(lp(r, B(ctx, r).rk[0]), o), n * E * 2});
            x.segs.push_back({L(u, V, n * E), at(lp(r, B(ctx, r).rv[0]), o), n * E * 2});
            xs.push_back(x);
          }
        }
      }
      WCK(run_phase(ctx, xs, tr, st));
      for (int r = 0; r < P; ++r) {
        const bool self = g.paper && !g.direct && pl.send[r] == r;
        sk[r] = self ? kteam(r) : lp(r, B(ctx, r).rk[0]);
        sv[r] = self ? vteam(r) : lp(r, B(ctx, r).rv[0]);
      }
    }

    for (int r = 0; r < P; ++r)
      if (local(ctx, r) && !ctx->dry) CK(cudaMemsetAsync(pdq(r, 0), 0, team * 4, st));

    const bool overlap = !ctx->emulated && !ctx->dry && R > 1;
    if (overlap) CK(cudaEventRecord(ctx->ev_a, st));
    for (int s = 0; s < R; ++s) {
      std::vector<Xfer> pk, dq;
      if (s < R - 1) {
        for (int r = 0; r < P; ++r) {
          const int dst = pl.next[r];
          const int s1 = (s + 1) & 1;
          Xfer x{1, WF_KIND_RING_QPKG, s, r, dst, pkg_team[r], {}};
          x.segs.push_back({pq(r, s), lp(dst, B(ctx, dst).pq[s1]), team * 2});
          x.segs.push_back({pdo(r, s), lp(dst, B(ctx, dst).pdo[s1]), team * 2});
          x.segs.push_back({plse(r, s), lp(dst, B(ctx, dst).plse[s1]), C * h * n * 4});
          x.segs.push_back({pds(r, s), lp(dst, B(ctx, dst).pdsum[s1]), C * h * n * 4});
          pk.push_back(x);
          Xfer y{1, WF_KIND_RING_DQ, s, r, dst, pkg_team[r], {}};
          y.segs.push_back({pdq(r, s), lp(dst, B(ctx, dst).pdq[s1]), team * 4});
          dq.push_back(y);
        }
        if (overlap) {
          // the package does not depend on step s: push it as soon as next released the slot
          if (s == 0) CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_a, 0));
          WCK(ipc_wait_ack(ctx, pl.next[ctx->rank], static_cast<uint32_t>(s), ctx->comm_stream));
          WCK(run_phase(ctx, pk, tr, ctx->comm_stream, kPhaseSend));
        }
      }
      for (int r = 0; r < P; ++r) {
        if (!local(ctx, r)) continue;
        RankBufs& b = B(ctx, r);
        BwdArgs a{};
        a.nq = C * g.n;
        a.nk = g.Bk;
        a.heads = g.h;
        a.causal = g.causal;
        a.qpos = units_table(g, pkg_team[r] * C, C);
        a.kpos = g.paper ? units_table(g, (pl.recv[r] / C) * C, C) : units_table(g, (r % C) * g.W, g.W);
        a.scale = 1.f / std::sqrt(static_cast<float>(g.d));
        a.scale_log2 = 1.4426950408889634f * a.scale;
        a.lse = plse(r, s);
        a.dsum = pds(r, s);
        a.stat_blk = g.n;
        a.dq_acc = pdq(r, s);
        a.dk_acc = b.dk_acc;
        a.dv_acc = b.dv_acc;
        a.dkv_accumulate = s > 0;
        if (P == 1) {  // one stationary block that is the whole K/V: write bf16 dK/dV directly
          a.dk_out = dK;
          a.dv_out = dV;
        }
        if (ctx->dry) continue;
        CUtensorMap tq, tk, tv, tdo;
        if (!make_tmap_rows(&tq, pq(r, s), a.nq, g.h, g.d) || !make_tmap_rows(&tk, sk[r], a.nk, g.h, g.d) ||
            !make_tmap_rows(&tv, sv[r], a.nk, g.h, g.d) || !make_tmap_rows(&tdo, pdo(r, s), a.nq, g.h, g.d))
          return fail(ctx, WF_ERR_ARG, "TMA map encode failed (alignment?)");
        WCK(dbg_bwd(ctx, a, pq(r, s), sk[r], sv[r], pdo(r, s), E));
        cudaEvent_t e0 = prof_begin(ctx, st);
        WCK(kcheck(ctx, launch_block_bwd(tq, tk, tv, tdo, a, g.d, st), "block_bwd"));
        prof_end(ctx, st, e0, ctx->ev_bwd);
      }
      if (s < R - 1) {
        if (overlap) {
          // dQ depends on step s: push it after the step; my package and dQ slots are free
          // once my kernel has read them and both sends have left (comm stream order), so
          // the release goes out from the comm stream after them; then wait for step s+1
          CK(cudaEventRecord(ctx->ev_b, st));
          CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->ev_b, 0));
          WCK(run_phase(ctx, dq, tr, ctx->comm_stream, kPhaseSend));
          WCK(ipc_ack(ctx, pl.last[ctx->rank], ctx->comm_stream));
          WCK(run_phase(ctx, pk, tr, ctx->comm_stream, kPhaseWait));
          WCK(run_phase(ctx, dq, tr, ctx->comm_stream, kPhaseWait));
          CK(cudaEventRecord(step_event(ctx, s), ctx->comm_stream));
          CK(cudaStreamWaitEvent(st, step_event(ctx, s), 0));
        } else {
          WCK(run_phase(ctx, pk, tr, st));
          WCK(run_phase(ctx, dq, tr, st));
        }
        std::vector<int> nt(P);
        for (int r = 0; r < P; ++r) nt[pl.next[r]] = pkg_team[r];
        pkg_team = nt;
      }
    }

    if (overlap && !(ctx->debug & WF_DEBUG_NO_TRANSFER)) ctx->ack_base[pl.next[ctx->rank]] += R - 1;

  }

  // return hop: dQ back to its home
  std::vector<float*> home(P, nullptr);
  if (R > 1) {
    std::vector<Xfer> xs;
    for (int r = 0; r < P; ++r) {
      const int dst = pl.next[r];
      Xfer x{1, WF_KIND_RET_DQ, R - 1, r, dst, pkg_team[r], {}};
      x.segs.push_back({pdq(r, R - 1), lp(dst, B(ctx, dst).home_dq), team * 4});
      xs.push_back(x);
    }
    WCK(run_phase(ctx, xs, tr, st));
    for (int r = 0; r < P; ++r) home[r] = lp(r, B(ctx, r).home_dq);
  } else {
    for (int r = 0; r < P; ++r) home[r] = pdq(r, 0);
  }

  // dK/dV (reading c11): every holder of a stationary block sends each unit's rows of its
  // fp32 partial straight to the unit's owner, who sums the replicas.  Holders of unit u:
  // paper regime, the C ranks whose stationary block is team(u); extension, the T ranks
  // whose slice contains u.  With peer memory the owner's sum kernel reads the holders'
  // accumulators in place (pull).
  auto first_unit = [&](int r) { return g.paper ? (pl.recv[r] / C) * C : (r % C) * g.W; };
  const int units_held = g.paper ? C : g.W;
  std::vector<std::vector<const float*>> kparts(P), vparts(P);
  {
    std::vector<std::vector<int>> holders(P);
    for (int r = 0; r < P; ++r)
      for (int u = first_unit(r); u < first_unit(r) + units_held; ++u) holders[u].push_back(r);
    auto slot_of = [&](int u, int r) {
      return static_cast<int>(std::find(holders[u].begin(), holders[u].end(), r) - holders[u].begin());
    };
    std::vector<Xfer> xs;
    for (int r = 0; r < P; ++r) {
      for (int u = first_unit(r); u < first_unit(r) + units_held; ++u) {
        if (u == r) continue;
        const int64_t o = static_cast<int64_t>(u - first_unit(r)) * n * E;
        const int64_t so = static_cast<int64_t>(slot_of(u, r)) * n * E;
        Xfer x{1, WF_KIND_REV_DKV, R, r, u, u, {}, ctx->ipc};
        x.segs.push_back({at(lp(r, B(ctx, r).dk_acc), o), at(lp(u, B(ctx, u).rev_k), so), n * E * 4});
        x.segs.push_back({at(lp(r, B(ctx, r).dv_acc), o), at(lp(u, B(ctx, u).rev_v), so), n * E * 4});
        xs.push_back(x);
      }
    }
    WCK(run_phase(ctx, xs, tr, st));
    for (int u = 0; u < P; ++u) {
      for (size_t i = 0; i < holders[u].size(); ++i) {
        const int r = holders[u][i];
        const int64_t o = static_cast<int64_t>(u - first_unit(r)) * n * E;
        const bool own = r == u;
        if (nt && !own) {  // no-transfer timing baseline: a local accumulator, same bytes
          kparts[u].push_back(lp(u, B(ctx, u).dk_acc));
          vparts[u].push_back(lp(u, B(ctx, u).dv_acc));
          continue;
        }
        kparts[u].push_back(own || ctx->ipc ? at(lp(r, B(ctx, r).dk_acc), o)
                                            : at(lp(u, B(ctx, u).rev_k), static_cast<int64_t>(i) * n * E));
        vparts[u].push_back(own || ctx->ipc ? at(lp(r, B(ctx, r).dv_acc), o)
                                            : at(lp(u, B(ctx, u).rev_v), static_cast<int64_t>(i) * n * E));
      }
    }
  }

  // dQ team reduce-scatter
  std::vector<std::vector<const float*>> qparts(P);
  if (C > 1) {
    std::vector<Xfer> xs;
    for (int r = 0; r < P; ++r) {
      const int t = r / C, j = r - t * C;
      for (int p = t * C; p < t * C + C; ++p) {
        if (p == r) continue;
        const int jp = p - t * C;
        const bool pushed = unitpipe && !last_unit_of(C, j, jp);
        Xfer x{1, WF_KIND_RS_DQ, R, r, p, p, {}, ctx->ipc && !pushed, pushed};
        x.segs.push_back({at(home[r], jp * n * E), at(lp(p, B(ctx, p).rsq), j * n * E), n * E * 4});
        xs.push_back(x);
      }
    }
    WCK(run_phase_after_pushes(ctx, xs, tr, st, unitpipe));
  }
  for (int r = 0; r < P; ++r) {
    const int j = r % C;
    for (int i = 0; i < C; ++i) {
      const int ri = (r / C) * C + i;
      const bool in_place = ctx->ipc && (!unitpipe || last_unit_of(C, i, j));
      qparts[r].push_back(i == j || nt ? at(home[r], i * n * E)
                          : in_place ? at(home[ri], j * n * E)
                                     : at(lp(r, B(ctx, r).rsq), i * n * E));
    }
  }
  if (ctx->dry) return WF_OK;
  for (int r = 0; r < P; ++r) {
    if (!local(ctx, r)) continue;
    const std::vector<const float*>* parts[3] = {&qparts[r], &kparts[r], &vparts[r]};
    bf16* outs[3] = {L(r, dQ, n * E), L(r, dK, n * E), L(r, dV, n * E)};
    for (int i = 0; i < 3; ++i) {
      if (P == 1 && i > 0) continue;  // dK/dV came out of the block kernel in bf16
      SumArgs s{};
      s.n = n * E;
      s.nparts = static_cast<int>(parts[i]->size());
      for (int k = 0; k < s.nparts; ++k) {
        s.parts[k] = (*parts[i])[k];
        WCK(dbg_check(ctx, s.parts[k], n * E * 4, "sum partial"));
      }
      s.out = outs[i];
      WCK(kcheck(ctx, launch_sum(s, st), "sum"));
    }
  }
  return join_comm(ctx, st);
}

wf_status new_ctx(int P, int C, wf_ctx** out, wf_ctx** tmp) {
  auto* ctx = new wf_ctx();
  *tmp = ctx;
  std::string err;
  if (!build_plan(P, C, &ctx->plan, &err)) {
    delete ctx;
    *tmp = nullptr;
    return fail(nullptr, WF_ERR_CONFIG, err);
  }
  *out = ctx;
  return WF_OK;
}

wf_status make_streams(wf_ctx* ctx) {
  CK(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ctx->ev_a, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_b, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ctx->ev_c, cudaEventDisableTiming));
  void* hf = nullptr;
  CK(cudaHostAlloc(&hf, 64, cudaHostAllocMapped));
  std::memset(hf, 0, 64);
  ctx->hfail = static_cast<volatile uint32_t*>(hf);
  void* df = nullptr;
  CK(cudaHostGetDevicePointer(&df, hf, 0));
  ctx->dfail = static_cast<uint32_t*>(df);
  return WF_OK;
}

// WF_ERR_COMM once a wait of an earlier call timed out (a peer stopped signalling): the
// failure is sticky, the context must be finalized.
wf_status comm_ok(wf_ctx* ctx) {
  if (ctx->comm) {  // the bootstrap communicator (wf_init): an asynchronous NCCL failure
    ncclResult_t ar = ncclSuccess;
    if (ncclCommGetAsyncError(ctx->comm, &ar) == ncclSuccess && ar != ncclSuccess && ar != ncclInProgress)
      return fail(ctx, WF_ERR_COMM, std::string("bootstrap communicator: ") + ncclGetErrorString(ar));
  }
  if (!ctx->hfail || ctx->hfail[0] == 0) return WF_OK;
  return fail(ctx, WF_ERR_COMM,
              "a peer did not signal within " + std::to_string(ctx->timeout_ns / 1000000000.0) +
                  " s (waited for count " + std::to_string(ctx->hfail[1]) + ", saw " + std::to_string(ctx->hfail[2]) +
                  "); finalize the context");
}

// begin a collective call: the failure check and the call sequence number (wf_qkv_proj's
// fused gather is consumed only by the call right after it)
wf_status begin_call(wf_ctx* ctx) {
  ++ctx->seq;
  return comm_ok(ctx);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// ====================================================================== C ABI
void wf_clear_ctxless_error() { g_ctxless_err.clear(); }

extern "C" {

wf_status wf_get_uid(wf_uid* out) {
  if (!out) return fail(nullptr, WF_ERR_ARG, "wf_get_uid: null");
  static_assert(sizeof(ncclUniqueId) <= sizeof(wf_uid), "uid size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, WF_ERR_COMM, ncclGetErrorString(r));
  std::memset(out, 0, sizeof(*out));
  std::memcpy(out->bytes, &id, sizeof(id));
  return WF_OK;
}

// Shared part of wf_init / wf_init_bootstrap: context, plan, streams.
static wf_status init_real(int P, int C, wf_topology topo, int rank, wf_ctx** out) {
  if (!out) return fail(nullptr, WF_ERR_ARG, "wf_init: null out");
  if (topo != WF_TOPO_COLLECT_INTRA && topo != WF_TOPO_P2P_INTRA) return fail(nullptr, WF_ERR_CONFIG, "bad topology");
  if (rank < 0 || rank >= P) return fail(nullptr, WF_ERR_CONFIG, "rank out of range");
  if (P > kMaxRanks) return fail(nullptr, WF_ERR_CONFIG, "P > 64 ranks is not supported by this build");
  wf_ctx* ctx = nullptr;
  wf_ctx* tmp = nullptr;
  WCK(new_ctx(P, C, &ctx, &tmp));
  ctx->rank = rank;
  ctx->ipc = P > 1;  // peer-memory transport between the P ranks
  wf_status s = make_streams(ctx);
  if (s != WF_OK) {
    g_ctxless_err = ctx->err;
    wf_finalize(ctx);
    return s;
  }
  *out = ctx;
  return WF_OK;
}

wf_status wf_init(int P, int C, wf_topology topo, int rank, const wf_uid* uid, wf_ctx** out) {
  wf_ctx* ctx = nullptr;
  WCK(init_real(P, C, topo, rank, &ctx));
  if (P > 1) {
    if (!uid) {
      wf_finalize(ctx);
      return fail(nullptr, WF_ERR_ARG, "wf_init: uid required when P > 1");
    }
    ncclUniqueId id;
    std::memcpy(&id, uid->bytes, sizeof(id));
    ncclResult_t r = ncclCommInitRank(&ctx->comm, P, id, rank);
    if (r != ncclSuccess) {
      wf_finalize(ctx);
      return fail(nullptr, WF_ERR_COMM, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
  }
  *out = ctx;
  return WF_OK;
}

wf_status wf_init_bootstrap(int P, int C, wf_topology topo, int rank, wf_allgather_fn allgather, void* user,
                            wf_ctx** out) {
  if (P > 1 && !allgather) return fail(nullptr, WF_ERR_ARG, "wf_init_bootstrap: allgather required when P > 1");
  wf_ctx* ctx = nullptr;
  WCK(init_real(P, C, topo, rank, &ctx));
  ctx->ag_fn = allgather;
  ctx->ag_user = user;
  *out = ctx;
  return WF_OK;
}

wf_status wf_init_emulated(int P, int C, wf_ctx** out) {
  if (!out) return fail(nullptr, WF_ERR_ARG, "wf_init_emulated: null out");
  wf_ctx* ctx = nullptr;
  wf_ctx* tmp = nullptr;
  WCK(new_ctx(P, C, &ctx, &tmp));
  ctx->emulated = true;
  wf_status s = make_streams(ctx);
  if (s != WF_OK) {
    g_ctxless_err = ctx->err;
    wf_finalize(ctx);
    return s;
  }
  *out = ctx;
  return WF_OK;
}

wf_status wf_set_timeout(wf_ctx* ctx, double seconds) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  if (!(seconds > 0)) return fail(ctx, WF_ERR_ARG, "wf_set_timeout: seconds must be > 0");
  ctx->timeout_ns = static_cast<uint64_t>(seconds * 1e9);
  return WF_OK;
}

wf_status wf_attn_fwd(wf_ctx* ctx, const void* Q, const void* K, const void* V, int64_t N, int heads, int head_dim,
                      int causal, void* O, float* LSE, void* stream) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  if (!Q || !K || !V || !O || !LSE) return fail(ctx, WF_ERR_ARG, "wf_attn_fwd: null pointer");
  if (!aligned16(Q) || !aligned16(K) || !aligned16(V) || !aligned16(O) || !aligned16(LSE))
    return fail(ctx, WF_ERR_ARG, "wf_attn_fwd: pointers must be 16-byte aligned");
  WCK(begin_call(ctx));
  Geo g;
  WCK(check_shape(ctx, N, heads, head_dim, causal, &g));
  WCK(ensure_ws(ctx, g));
  return forward(ctx, g, static_cast<const bf16*>(Q), static_cast<const bf16*>(K), static_cast<const bf16*>(V),
                 static_cast<bf16*>(O), LSE, static_cast<cudaStream_t>(stream));
}

wf_status wf_qkv_proj(wf_ctx* ctx, const void* X, const void* W, int64_t N, int hidden, int heads, int head_dim,
                      int causal, void* Q, void* K, void* V, void* stream) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  if (!X || !W || !Q || !K || !V) return fail(ctx, WF_ERR_ARG, "wf_qkv_proj: null pointer");
  for (const void* p : {X, W, static_cast<const void*>(Q), static_cast<const void*>(K), static_cast<const void*>(V)})
    if (!aligned16(p)) return fail(ctx, WF_ERR_ARG, "wf_qkv_proj: pointers must be 16-byte aligned");
  WCK(begin_call(ctx));
  Geo g;
  WCK(check_shape(ctx, N, heads, head_dim, causal, &g));
  const int64_t n = g.n, E = g.E;
  if (hidden <= 0 || hidden % 64 || E % 128 || n % 128)
    return fail(ctx, WF_ERR_CONFIG, "wf_qkv_proj: hidden % 64, (heads*head_dim) % 128 and (N/P) % 128 must be 0");
  WCK(ensure_ws(ctx, g));
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int P = g.P, C = g.C;
  const int bn = E % 256 == 0 ? 256 : 128;
  GemmArgs shape{};
  shape.M = static_cast<int>(n);
  shape.N = static_cast<int>(3 * E);
  shape.split = static_cast<int>(E);
  const bool pair = gemm_pair_ok(shape, 0, 0);
  CUtensorMap tw;
  if (!make_tmap_2d(&tw, W, 3 * E, hidden, pair ? 128 : bn))
    return fail(ctx, WF_ERR_ARG, "wf_qkv_proj: TMA map encode failed");
  // fused gather: the epilogue writes straight into the team buffers (peer memory or, emulated,
  // the virtual ranks' workspaces)
  bool fuse = C > 1 && !(ctx->debug & WF_DEBUG_NO_TRANSFER);
  if (fuse && C + 2 > WF_GEMM_MAX_DST) fuse = false;
  if (fuse && ctx->ipc) WCK(ipc_barrier(ctx, st));  // every peer is done with its team buffers
  auto lp = [&](int r, bf16* p) { return addressable(ctx, r) ? p : nullptr; };
  {
    const int64_t nr = ctx->emulated ? P : 1;
    dbg_begin(ctx, {{X, nr * n * hidden * 2}, {W, 3 * E * hidden * 2}, {Q, nr * n * E * 2}, {K, nr * n * E * 2},
                    {V, nr * n * E * 2}});
  }
  for (int r = 0; r < P; ++r) {
    if (!local(ctx, r)) continue;
    const int64_t ro = ctx->emulated ? r : 0;
    GemmArgs ga{};
    ga.M = static_cast<int>(n);
    ga.N = static_cast<int>(3 * E);
    ga.K = hidden;
    ga.split = static_cast<int>(E);
    ga.ld = E;
    bf16* outs[3] = {static_cast<bf16*>(Q) + ro * n * E, static_cast<bf16*>(K) + ro * n * E,
                     static_cast<bf16*>(V) + ro * n * E};
    for (int part = 0; part < 3; ++part) {
      ga.out[part][0] = outs[part];
      ga.ndst[part] = 1;
    }
    if (fuse) {
      const int t = r / C, j = r - t * C;
      auto add = [&](int part, bf16* p) -> bool {
        if (!p || ga.ndst[part] >= WF_GEMM_MAX_DST) return false;
        ga.out[part][ga.ndst[part]++] = p;
        return true;
      };
      bool ok = true;
      for (int p = t * C; p < t * C + C; ++p) {  // Alg. 1 l.1: member-major team tensors
        ok = ok && add(0, at(lp(p, B(ctx, p).qt), j * n * E));
        if (g.paper && !g.direct) {
          ok = ok && add(1, at(lp(p, B(ctx, p).kt), j * n * E));
          ok = ok && add(2, at(lp(p, B(ctx, p).vt), j * n * E));
        }
      }
      if (!g.paper || g.direct) {  // unit r goes to every rank whose first K/V block holds it
        for (int p = 0; p < P; ++p) {
          const int kf = g.paper ? (ctx->plan.recv[p] / C) * C : (p % C) * g.W;
          const int kc = g.paper ? C : g.W;
          if (r < kf || r >= kf + kc) continue;
          const int64_t off = static_cast<int64_t>(r - kf) * n * E;
          ok = ok && add(1, at(lp(p, B(ctx, p).rk[0]), off));
          ok = ok && add(2, at(lp(p, B(ctx, p).rv[0]), off));
        }
      }
      if (!ok) return fail(ctx, WF_ERR_CONFIG, "wf_qkv_proj: too many gather destinations");
    }
    for (int part = 0; part < 3; ++part)
      for (int i = 0; i < ga.ndst[part]; ++i) WCK(dbg_check(ctx, ga.out[part][i], n * E * 2, "projection output"));
    CUtensorMap tx;
    if (!make_tmap_2d(&tx, static_cast<const bf16*>(X) + ro * n * hidden, n, hidden, 128))
      return fail(ctx, WF_ERR_ARG, "wf_qkv_proj: TMA map encode failed");
    WCK(kcheck(ctx, pair ? launch_gemm_pair(tx, tw, ga, 0, 0, st) : launch_gemm(tx, tw, ga, bn, st), "qkv_gemm"));
  }
  if (fuse) {
    ctx->proj_seq = ctx->seq;
    ctx->proj_q = Q;
    ctx->proj_k = K;
    ctx->proj_v = V;
    const int64_t key[4] = {g.N, g.h, g.d, g.causal};
    std::copy(key, key + 4, ctx->proj_key);
  }
  return WF_OK;
}

wf_status wf_attn_bwd(wf_ctx* ctx, const void* dO, const void* Q, const void* K, const void* V, const void* O,
                      const float* LSE, int64_t N, int heads, int head_dim, int causal, void* dQ, void* dK, void* dV,
                      void* stream) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  if (!dO || !Q || !K || !V || !O || !LSE || !dQ || !dK || !dV) return fail(ctx, WF_ERR_ARG, "wf_attn_bwd: null pointer");
  for (const void* p : {dO, Q, K, V, O, static_cast<const void*>(LSE), static_cast<const void*>(dQ),
                        static_cast<const void*>(dK), static_cast<const void*>(dV)})
    if (!aligned16(p)) return fail(ctx, WF_ERR_ARG, "wf_attn_bwd: pointers must be 16-byte aligned");
  WCK(begin_call(ctx));
  Geo g;
  WCK(check_shape(ctx, N, heads, head_dim, causal, &g));
  WCK(ensure_ws(ctx, g));
  return backward(ctx, g, static_cast<const bf16*>(dO), static_cast<const bf16*>(Q), static_cast<const bf16*>(K),
                  static_cast<const bf16*>(V), static_cast<const bf16*>(O), LSE, static_cast<bf16*>(dQ),
                  static_cast<bf16*>(dK), static_cast<bf16*>(dV), static_cast<cudaStream_t>(stream));
}

static wf_status copy_trace(const std::vector<wf_event>& a, const std::vector<wf_event>& b, wf_event* buf, size_t cap,
                            size_t* n_out) {
  const size_t n = a.size() + b.size();
  if (n_out) *n_out = n;
  if (buf) {
    size_t k = 0;
    for (const auto& e : a)
      if (k < cap) buf[k++] = e;
    for (const auto& e : b)
      if (k < cap) buf[k++] = e;
  }
  return WF_OK;
}

wf_status wf_get_trace(wf_ctx* ctx, wf_event* buf, size_t cap, size_t* n_out) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  return copy_trace(ctx->trace_fwd, ctx->trace_bwd, buf, cap, n_out);
}

wf_status wf_workspace_bytes(int P, int C, int64_t N, int heads, int head_dim, int causal, size_t* bytes) {
  if (!bytes) return fail(nullptr, WF_ERR_ARG, "wf_workspace_bytes: null output");
  wf_ctx* ctx = nullptr;
  wf_ctx* tmp = nullptr;
  WCK(new_ctx(P, C, &ctx, &tmp));
  std::unique_ptr<wf_ctx> hold(ctx);
  ctx->dry = true;
  Geo g;
  wf_status s = check_shape(ctx, N, heads, head_dim, causal, &g);
  if (s != WF_OK) return fail(nullptr, s, ctx->err);
  RankBufs b{};
  CarveList items;
  carve_rank(g, b, items, false);  // real mode (peer memory) carve
  *bytes = carve_total(items);
  return WF_OK;
}

wf_status wf_plan_trace_sched(int P, int C, int64_t N, int heads, int head_dim, int rank, int sched, wf_event* buf,
                              size_t cap, size_t* n_out) {
  wf_ctx* ctx = nullptr;
  wf_ctx* tmp = nullptr;
  WCK(new_ctx(P, C, &ctx, &tmp));
  std::unique_ptr<wf_ctx> hold(ctx);
  ctx->dry = true;
  ctx->dry_rank = rank;
  ctx->sched = sched;
  Geo g;
  // full-mask geometry (the trace is mask independent)
  wf_status s = check_shape(ctx, N, heads, head_dim, 0, &g);
  if (s != WF_OK) return fail(nullptr, s, ctx->err);
  ensure_ws(ctx, g);
  s = forward(ctx, g, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  if (s == WF_OK) s = backward(ctx, g, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr);
  if (s != WF_OK) return fail(nullptr, s, ctx->err);
  return copy_trace(ctx->trace_fwd, ctx->trace_bwd, buf, cap, n_out);
}

wf_status wf_plan_trace(int P, int C, int64_t N, int heads, int head_dim, int rank, wf_event* buf, size_t cap,
                        size_t* n_out) {
  return wf_plan_trace_sched(P, C, N, heads, head_dim, rank, WF_SCHED_GATHER_SHUFFLE, buf, cap, n_out);
}

wf_status wf_set_schedule(wf_ctx* ctx, int sched) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  if (sched != WF_SCHED_GATHER_SHUFFLE && sched != WF_SCHED_DIRECT_PULL)
    return fail(ctx, WF_ERR_CONFIG, "wf_set_schedule: unknown schedule");
  ctx->sched = sched;
  ++ctx->seq;  // a pending fused gather used the old layout
  return WF_OK;
}

wf_status wf_plan(int P, int C, int rank, int32_t out[6]) {
  Plan p;
  std::string err;
  if (!build_plan(P, C, &p, &err)) return fail(nullptr, WF_ERR_CONFIG, err);
  if (rank < 0 || rank >= P || !out) return fail(nullptr, WF_ERR_ARG, "wf_plan: bad rank/out");
  out[0] = p.send[rank];
  out[1] = p.recv[rank];
  out[2] = p.next[rank];
  out[3] = p.last[rank];
  out[4] = p.R;
  out[5] = p.paper ? 0 : 1;
  return WF_OK;
}

wf_status wf_shard_ranges(int P, int rank, int64_t N, int causal, int64_t ranges[4]) {
  if (P < 1 || rank < 0 || rank >= P || !ranges) return fail(nullptr, WF_ERR_ARG, "wf_shard_ranges: bad args");
  if (causal) {
    if (N % (2 * P)) return fail(nullptr, WF_ERR_CONFIG, "zigzag needs 2P | N");
    const int64_t c = N / (2 * P);
    ranges[0] = rank * c;
    ranges[1] = (rank + 1) * c;
    ranges[2] = (2LL * P - 1 - rank) * c;
    ranges[3] = (2LL * P - rank) * c;
  } else {
    if (N % P) return fail(nullptr, WF_ERR_CONFIG, "naive split needs P | N");
    const int64_t n = N / P;
    ranges[0] = rank * n;
    ranges[1] = (rank + 1) * n;
    ranges[2] = ranges[3] = ranges[1];
  }
  return WF_OK;
}

int64_t wf_kernel_launches(const wf_ctx* ctx) { return ctx ? ctx->launches : 0; }

wf_status wf_phase_times(wf_ctx* ctx, double* ms_by_kind, int n) {
  if (!ctx || !ms_by_kind) return fail(ctx, WF_ERR_ARG, "wf_phase_times: null");
  CK(cudaDeviceSynchronize());
  for (int i = 0; i < n; ++i) ms_by_kind[i] = 0;
  for (auto& pr : ctx->ev_phase) {
    float t = 0;
    CK(cudaEventElapsedTime(&t, pr.second.first, pr.second.second));
    if (pr.first >= 0 && pr.first < n) ms_by_kind[pr.first] += t;
    ctx->ev_pool.push_back(pr.second.first);
    ctx->ev_pool.push_back(pr.second.second);
  }
  ctx->ev_phase.clear();
  return WF_OK;
}

wf_status wf_set_debug(wf_ctx* ctx, int flags) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  ctx->debug = flags;
  return WF_OK;
}

wf_status wf_set_profiling(wf_ctx* ctx, int on) {
  if (!ctx) return fail(nullptr, WF_ERR_ARG, "null ctx");
  ctx->profiling = on != 0;
  return WF_OK;
}

wf_status wf_kernel_times(wf_ctx* ctx, double out[4]) {
  if (!ctx || !out) return fail(ctx, WF_ERR_ARG, "wf_kernel_times: null");
  CK(cudaDeviceSynchronize());
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>>* lists[2] = {&ctx->ev_fwd, &ctx->ev_bwd};
  for (int i = 0; i < 2; ++i) {
    double ms = 0;
    for (auto& pr : *lists[i]) {
      float t = 0;
      CK(cudaEventElapsedTime(&t, pr.first, pr.second));
      ms += t;
      ctx->ev_pool.push_back(pr.first);
      ctx->ev_pool.push_back(pr.second);
    }
    out[i] = ms;
    out[2 + i] = static_cast<double>(lists[i]->size());
    lists[i]->clear();
  }
  return WF_OK;
}

const char* wf_last_error(const wf_ctx* ctx) {
  if (ctx) return ctx->err.c_str();
  if (!g_ctxless_err.empty()) return g_ctxless_err.c_str();
  return wf_static_error();
}

wf_status wf_finalize(wf_ctx* ctx) {
  if (!ctx) return WF_OK;
  if (ctx->ws) {
    cudaDeviceSynchronize();
    if (ctx->ipc && ctx->comm_stream && !ctx->peer_base.empty() && comm_ok(ctx) == WF_OK) {
      // collective: peers may still pull from this workspace -- free it after every rank
      // has finished its last call (a rank that never joins ends the wait at the timeout)
      if (ipc_barrier(ctx, ctx->comm_stream) == WF_OK) cudaStreamSynchronize(ctx->comm_stream);
    }
    for (size_t r = 0; r < ctx->peer_base.size(); ++r)
      if (static_cast<int>(r) != ctx->rank && ctx->peer_base[r]) cudaIpcCloseMemHandle(ctx->peer_base[r]);
    cudaFree(ctx->ws);
  }
  for (cudaEvent_t e : ctx->ev_step) cudaEventDestroy(e);
  for (cudaEvent_t e : ctx->ev_src) cudaEventDestroy(e);
  if (ctx->ev_c) cudaEventDestroy(ctx->ev_c);
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
  for (auto& pr : ctx->ev_fwd) ctx->ev_pool.push_back(pr.first), ctx->ev_pool.push_back(pr.second);
  for (auto& pr : ctx->ev_bwd) ctx->ev_pool.push_back(pr.first), ctx->ev_pool.push_back(pr.second);
  for (auto& pr : ctx->ev_phase) ctx->ev_pool.push_back(pr.second.first), ctx->ev_pool.push_back(pr.second.second);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->hfail) cudaFreeHost(const_cast<uint32_t*>(ctx->hfail));
  delete ctx;
  return WF_OK;
}

}  // extern "C"
