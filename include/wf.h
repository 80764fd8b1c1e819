/* wf.h -- C ABI of the B200-native WallFacer multi-ring attention library (libwf.so).
 *
 * WallFacer (arXiv 2407.00611) shards one sequence of N tokens over P GPUs, groups
 * them into P/C teams of C (§3.2.1), team-gathers Q/K/V, passes K/V
 * blocks along C^2 sub-rings of length P/C^2 (Alg. 1; Alg. 2/3,
 * PAPER.md:263-292) and merges the C partial (O, lse) results of a team with an
 * LSE-weighted reduce-scatter (Alg. 1 l.11).  The backward keeps K/V
 * and dK/dV stationary and circulates the queries with dQ.
 * At C = 1 the same calls are plain Ring Attention.
 *
 * Conventions (all calls):
 *  - One process per GPU.  All pointers are DEVICE pointers owned by the caller
 *    unless stated; nothing is freed or retained by the library after a call returns
 *    except the context's own workspace.
 *  - Tensors are contiguous [tokens, heads, head_dim] bf16 (B = 1),
 *    rows 16-byte aligned.  LSE is fp32 [heads, tokens], natural log (reading c16).
 *  - Causal inputs are the caller's ZIGZAG shard: rank r passes chunk r followed by
 *    chunk 2P-1-r of the 2P equal chunks (reading c13); full-mask inputs
 *    are the contiguous shard [r N/P, (r+1) N/P).  wf_shard_ranges
 *    returns these ranges.
 *  - Work is enqueued on `stream` and the call returns after enqueue; internal streams
 *    are joined back into `stream` before return.  Every rank calls collectively with
 *    identical (N, heads, head_dim, causal).
 *  - Errors: every call returns a wf_status; wf_last_error(ctx) gives the text.
 *    WF_ERR_CONFIG: invalid (P, C) or unsupported shape (head_dim not in {64, 72, 128};
 *    N not a multiple of 128 P (full) or 256 P (causal)).  WF_ERR_ARG: null or
 *    misaligned pointer.  WF_ERR_CUDA: a CUDA failure.  WF_ERR_COMM: a bootstrap
 *    failure, or -- asynchronously -- a peer that stopped signalling: a wait of an
 *    earlier call timed out (wf_set_timeout, default 30 s), so the next wf_attn_fwd /
 *    wf_attn_bwd / wf_qkv_proj returns WF_ERR_COMM (sticky).  After WF_ERR_CUDA or
 *    WF_ERR_COMM the context should be finalized.  (Mirrors SPEC.md:524 exit codes 0/1/2.)
 */
#ifndef WF_H_
#define WF_H_
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct wf_ctx wf_ctx; /* opaque: plan, communicators, workspace, streams, trace */

typedef enum {
  WF_OK = 0,
  WF_ERR_NUMERIC = 1, /* harness-level only (tolerance / trace mismatch) */
  WF_ERR_CONFIG = 2,
  WF_ERR_ARG = 3,
  WF_ERR_CUDA = 4,
  WF_ERR_COMM = 5
} wf_status;

typedef enum {
  WF_TOPO_COLLECT_INTRA = 0, /* teams contiguous in rank: Alg. 2's placement */
  WF_TOPO_P2P_INTRA = 1      /* accepted; identical on one NVSwitch node      */
} wf_topology;

/* Opaque 128-byte id wrapping an ncclUniqueId.  Rank 0 calls wf_get_uid and the
 * caller broadcasts the bytes (e.g. torch.distributed) to every rank before wf_init. */
typedef struct {
  uint8_t bytes[128];
} wf_uid;

/* One CommTrace record (SURVEY.md §8(c) "Oracle schedule simulator"): pass 0 = forward,
 * 1 = backward; kind is a WF_KIND_* value; step -1 gathers / init shuffle, s in
 * [0, R-2] ring hop after compute step s, R-1 the dQ return hop, R post-loop reductions;
 * block = team block, team, or unit id (by kind); bytes on the wire.  Only messages
 * with src != dst are recorded. */
typedef struct {
  int32_t pass, kind, step, src, dst, block;
  int64_t bytes;
} wf_event;

enum {
  WF_KIND_AG_Q = 0, WF_KIND_AG_KV, WF_KIND_INIT_KV, WF_KIND_SLICE_KV, WF_KIND_RING_KV, WF_KIND_RS_O,
  WF_KIND_RS_LSE, WF_KIND_AG_QDO, WF_KIND_AG_STATS, WF_KIND_RING_QPKG, WF_KIND_RING_DQ, WF_KIND_RET_DQ,
  WF_KIND_REV_DKV, WF_KIND_RS_DKV, WF_KIND_RS_DQ, WF_KIND_COUNT
};

/* Rank 0: create the NCCL unique id of a new context.  out: host memory. */
wf_status wf_get_uid(wf_uid* out);

/* Create this rank's context: validates (P, C) (reading c2: C | P and, when C^2 <= P,
 * C^2 | P; C^2 > P is the extension regime with R = 1), builds the plan (Alg. 2/3),
 * creates the bootstrap NCCL communicator on the current CUDA device (used only to
 * exchange the workspaces' CUDA IPC handles; every message of the schedule then moves
 * over peer memory).  uid: host memory, the same bytes on every rank; may
 * be NULL when P == 1.  out: receives the context.  P <= 64. */
wf_status wf_init(int P, int C, wf_topology topo, int rank, const wf_uid* uid, wf_ctx** out);

/* Host all-gather supplied by the caller: every rank passes `bytes` bytes at `in` (host
 * memory) and receives the P contributions rank-major at `out` (P * bytes); blocking,
 * collective; returns 0 on success.  `user` is passed through. */
typedef int (*wf_allgather_fn)(const void* in, void* out, size_t bytes, void* user);

/* As wf_init, with the IPC-handle exchange done by the caller's host collective instead of
 * NCCL (e.g. torch.distributed over gloo).  Needs no NCCL communicator, so several ranks
 * may share one GPU (each its own process): the real peer-memory transport can be tested
 * on a single device.  allgather may be NULL when P == 1; it is called from inside the
 * first wf_attn_fwd / wf_attn_bwd / wf_qkv_proj of a new shape (collective). */
wf_status wf_init_bootstrap(int P, int C, wf_topology topo, int rank, wf_allgather_fn allgather, void* user,
                            wf_ctx** out);

/* Timeout of every inter-rank wait of this context (default 30 s).  A wait that times out
 * is reported as WF_ERR_COMM by the next call (see Errors).  seconds > 0. */
wf_status wf_set_timeout(wf_ctx* ctx, double seconds);

/* Single-GPU emulation of all P ranks (test/bench aid): the same schedule, block
 * kernels and trace, with every message a device-local copy.  In this mode every
 * tensor argument of wf_attn_fwd / wf_attn_bwd addresses the P rank shards
 * concatenated rank-major: [P][N/P, heads, head_dim] (LSE: [P][heads, N/P]). */
wf_status wf_init_emulated(int P, int C, wf_ctx** out);

/* Forward (Alg. 1): Q, K, V bf16 [N/P, heads, head_dim] (this rank's shard) ->
 * O bf16 [N/P, heads, head_dim], LSE fp32 [heads, N/P]. */
wf_status wf_attn_fwd(wf_ctx* ctx, const void* Q, const void* K, const void* V, int64_t N, int heads,
                      int head_dim, int causal, void* O, float* LSE, void* stream);

/* QKV projection fused with the team all-gather (Alg. 1 l.1
 * "AllGather_QKVmatmul").  X bf16 [N/P, hidden]
 * (this rank's shard of the layer input), W bf16 [3 heads head_dim, hidden] (row-major,
 * the stacked W_q; W_k; W_v of nn.Linear, replicated on every rank) ->
 * Q, K, V bf16 [N/P, heads, head_dim] = X W^T split in three.  With C > 1 the GEMM's
 * epilogue also stores every output tile into the team members' gathered buffers (peer
 * memory; in the extension regime K/V go to the ranks whose slice holds this unit), so
 * the next wf_attn_fwd on this context with these Q, K, V skips the gather copies (its
 * CommTrace is unchanged: the same messages, moved by the epilogue).  Emulated mode:
 * X [P][N/P, hidden], outputs [P][N/P, heads, head_dim].  hidden: multiple of 64;
 * N/P: multiple of 128; heads * head_dim: multiple of 128.  WF_ERR_CONFIG otherwise. */
wf_status wf_qkv_proj(wf_ctx* ctx, const void* X, const void* W, int64_t N, int hidden, int heads, int head_dim,
                      int causal, void* Q, void* K, void* V, void* stream);

/* Backward: given dO and the forward's Q, K, V, O, LSE (same
 * shapes as wf_attn_fwd) -> dQ, dK, dV bf16 [N/P, heads, head_dim]. */
wf_status wf_attn_bwd(wf_ctx* ctx, const void* dO, const void* Q, const void* K, const void* V, const void* O,
                      const float* LSE, int64_t N, int heads, int head_dim, int causal, void* dQ, void* dK,
                      void* dV, void* stream);

/* Copy the CommTrace of the last forward + backward of this rank (all ranks in
 * emulated mode) into buf (host memory, cap records).  n_out: records available. */
wf_status wf_get_trace(wf_ctx* ctx, wf_event* buf, size_t cap, size_t* n_out);

/* Host-only: the trace this library will emit for (P, C, N, heads, head_dim) and one
 * rank (rank = -1: all ranks), forward and backward, without a GPU or a context.
 * Same record semantics as wf_get_trace. */
wf_status wf_plan_trace(int P, int C, int64_t N, int heads, int head_dim, int rank, wf_event* buf, size_t cap,
                        size_t* n_out);

/* Host-only: bytes of device workspace one rank of a real (peer-memory) (P, C) context
 * allocates for this shape with the default schedule, sized by regime: team buffers,
 * K/V receive slots (two for a ring, one at R = 1, none at P = 1), fp32 state and
 * dQ/dK/dV accumulators, receive slots only where partials are pushed.  This is the library's counterpart of the paper's 3CA activation
 * term (Eq. 7).  WF_ERR_CONFIG on an invalid shape, WF_ERR_ARG if
 * bytes is null. */
wf_status wf_workspace_bytes(int P, int C, int64_t N, int heads, int head_dim, int causal, size_t* bytes);

/* Schedule variants (SURVEY.md §8(a) "Schedule variants", reading c21).  Both compute the
 * same result; they differ in how the paper regime's first K/V block reaches a rank:
 * WF_SCHED_GATHER_SHUFFLE (default, the paper's Alg. 1 l.1-2): team all-gather of K/V,
 * then the init shuffle of the team block to init_send (AG_KV + INIT_KV messages);
 * WF_SCHED_DIRECT_PULL: every unit of the block team(init_recv) comes straight from its
 * owner (SLICE_KV messages, as in the extension regime), one hop instead of two; with
 * R = 1 the step is then unit-pipelined like the extension regime.  Set before the first
 * wf_attn_fwd of a shape; the extension regime and C = 1 are unaffected. */
#define WF_SCHED_GATHER_SHUFFLE 0
#define WF_SCHED_DIRECT_PULL 1
wf_status wf_set_schedule(wf_ctx* ctx, int sched);
wf_status wf_plan_trace_sched(int P, int C, int64_t N, int heads, int head_dim, int rank, int sched, wf_event* buf,
                              size_t cap, size_t* n_out);

/* Host-only: the plan of one rank: out[0..5] = {init_send, init_recv, next, last, R, regime}
 * (regime 0 = paper, 1 = extension). */
wf_status wf_plan(int P, int C, int rank, int32_t out[6]);

/* Host-only: global token ranges of rank's shard: ranges[0..3] =
 * {a0, a1, b0, b1}, the shard being [a0, a1) followed by [b0, b1) (b0 == b1 when full). */
wf_status wf_shard_ranges(int P, int rank, int64_t N, int causal, int64_t ranges[4]);

/* Timing aid: number of kernels this context launched since creation. */
int64_t wf_kernel_launches(const wf_ctx* ctx);

/* Timing aid (bench): when on != 0, CUDA events are recorded on the launching stream
 * around every block-forward and block-backward kernel.  wf_kernel_times synchronizes
 * and returns the summed device milliseconds and launch counts since profiling was
 * enabled (out[0] fwd ms, out[1] bwd ms, out[2] fwd launches, out[3] bwd launches). */
wf_status wf_set_profiling(wf_ctx* ctx, int on);
wf_status wf_kernel_times(wf_ctx* ctx, double out[4]);
/* With profiling on: device milliseconds spent in each message phase since the last call,
 * summed by WF_KIND_* (ms_by_kind[0..n)), measured by events on the phase's stream. */
wf_status wf_phase_times(wf_ctx* ctx, double* ms_by_kind, int n);

/* Measurement aid (bench): flags = WF_DEBUG_NO_TRANSFER skips every inter-rank transfer
 * (the kernels run on whatever the receive buffers hold, the trace is still recorded), so
 * T(no transfer) / T gives the exposed-communication fraction with identical kernels.
 * Results are garbage in that mode. */
#define WF_DEBUG_NO_TRANSFER 1
wf_status wf_set_debug(wf_ctx* ctx, int flags);

/* Debug aid: record clock64() stamps of the block kernels' warp roles for CTA (cta, head 0)
 * of every launch (cta < 0: off); read n words after the launches (layout: slot
 * (role * 1024 + tile) * 8 + event, see csrc/attn_fwd.cu / attn_bwd.cu). */
wf_status wf_debug_timeline(int cta);
wf_status wf_debug_timeline_read(unsigned long long* out, size_t n);

/* Last error text of ctx (or of the last context-less call when ctx is NULL). */
const char* wf_last_error(const wf_ctx* ctx);

/* Destroy the context: frees workspace, communicators, streams.  Collective over the P
 * ranks of a real (peer-memory) context: the workspace is freed only after every rank has
 * finished its last call, since peers read it in place. */
wf_status wf_finalize(wf_ctx* ctx);

/* ---- per-step kernels, exported for parity tests of one ring step ---------------
 * wf_block_fwd: PAPER.md:183 forward_iteration on one device.  q [nq, heads, D],
 * k/v [nk, heads, D] bf16; positions: row r of q sits at global token
 * qstart[r / chunk] + r % chunk (likewise k); chunk multiple of 128 (ignored unless
 * causal).  o_in/lse_in: optional fp32 state (NULL = empty state, lse = -inf).
 * Writes fp32 o_out (if non-NULL), bf16 o_bf16 (if non-NULL) and lse_out [heads, nq]. */
wf_status wf_block_fwd(const void* q, const void* k, const void* v, int nq, int nk, int heads, int head_dim,
                       int causal, int chunk, const int32_t* qstart, int nqchunks, const int32_t* kstart,
                       int nkchunks, const float* o_in, const float* lse_in, float* o_out, void* o_bf16,
                       float* lse_out, void* stream);

/* wf_gemm_bf16: Y = A B^T on the tensor cores (the projection GEMM of wf_qkv_proj),
 * A bf16 [M, K], B bf16 [N, K], Y bf16 [M, N], all row-major, fp32 accumulation.
 * M multiple of 128, N of 128, K of 64 (WF_ERR_CONFIG otherwise); 16-byte aligned. */
wf_status wf_gemm_bf16(const void* A, const void* B, int M, int N, int K, void* Y, void* stream);
/* General layouts: Y[m, n] = sum_k A(m, k) B(n, k) with A stored [M, K] (a_mn = 0) or
 * [K, M] (a_mn = 1), B stored [N, K] (b_mn = 0) or [K, N] (b_mn = 1): the backward
 * products dX = dY W (a_mn 0, b_mn 1) and dW = dY^T X (a_mn 1, b_mn 1) of a projection. */
wf_status wf_gemm_bf16_t(const void* A, int a_mn, const void* B, int b_mn, int M, int N, int K, void* Y,
                         void* stream);

/* ---- the other operators of a WallFacer Transformer layer (
 * P:199 "finalized after a standard LayerNorm and FeedForward layer process", driven by
 * paper_2407_00611_b200/layer.py; reading c22) ----
 * All bf16 row-major device buffers, 16-byte aligned; status as above.
 * wf_layernorm_fwd: y = (x - mean) rstd w + b per row (nn.LayerNorm, affine), mean and
 *   rstd = 1/sqrt(var + eps) fp32 [rows] out (var biased).  hidden % 8 == 0, <= 8192.
 * wf_layernorm_bwd: with xhat = (x - mean) rstd, g = w o dy:
 *   dx = rstd (g - mean(g) - xhat mean(g o xhat)) (+ dres if non-NULL: the residual
 *   branch's gradient); dw += sum_rows dy o xhat, db += sum_rows dy (fp32 [hidden],
 *   accumulated: zero them first).
 * wf_gelu_fwd: h = u Phi(u) elementwise (exact erf GELU, the FeedForward activation; erf
 *   evaluated to |error| <= 1.5e-7, Abramowitz & Stegun 7.1.26); n elements, n % 8 == 0.
 * wf_gelu_bwd: du = dh o (Phi(u) + u phi(u)).
 * wf_add_bf16: y = a + b (n elements, n % 8 == 0).
 * wf_pack3_bf16: y [rows, 3E] = [a | b | c] (a, b, c [rows, E]). */
wf_status wf_layernorm_fwd(const void* x, const void* w, const void* b, int64_t rows, int hidden, float eps, void* y,
                           float* mean, float* rstd, void* stream);
wf_status wf_layernorm_bwd(const void* dy, const void* x, const void* w, const float* mean, const float* rstd,
                           const void* dres, int64_t rows, int hidden, void* dx, float* dw, float* db, void* stream);
wf_status wf_gelu_fwd(const void* u, int64_t n, void* h, void* stream);
wf_status wf_gelu_bwd(const void* dh, const void* u, int64_t n, void* du, void* stream);
wf_status wf_add_bf16(const void* a, const void* b, int64_t n, void* y, void* stream);
wf_status wf_pack3_bf16(const void* a, const void* b, const void* c, int64_t rows, int E, void* y, void* stream);

/* wf_block_bwd: PAPER.md:203 one flash-attention backward step: the K/V block
 * (stationary) against query rows q with dO, final LSE and D = rowsum(dO o O) [heads, nq].
 * dq_acc fp32 [nq, heads, D] is accumulated (+=) atomically; dk_acc/dv_acc fp32
 * [nk, heads, D] are accumulated when accumulate != 0, else overwritten. */
wf_status wf_block_bwd(const void* q, const void* k, const void* v, const void* dO, const float* lse,
                       const float* dsum, int nq, int nk, int heads, int head_dim, int causal, int chunk,
                       const int32_t* qstart, int nqchunks, const int32_t* kstart, int nkchunks, float* dq_acc,
                       float* dk_acc, float* dv_acc, int accumulate, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* WF_H_ */
