// blocks_api.cu -- TMA map encoding and the exported per-step kernel entry points
// (wf_block_fwd / wf_block_bwd of include/wf.h).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/wf.h"
#include "common.h"
#include "internal.h"

namespace wf {

namespace {
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}
}  // namespace

bool make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int heads, int D) {
  return make_tmap_rows_box(map, base, rows, heads, D, WF_TILE);
}

bool make_tmap_rows_box(CUtensorMap* map, const void* base, int64_t rows, int heads, int D, int box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(heads), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 2, static_cast<cuuint64_t>(heads) * D * 2};
  cuuint32_t box[3] = {64, 1, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_f32_rows(CUtensorMap* map, const void* base, int64_t rows, int heads, int D) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(D), static_cast<cuuint64_t>(heads), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(D) * 4, static_cast<cuuint64_t>(heads) * D * 4};
  cuuint32_t box[3] = {32, 1, 32};  // one warp's 32 query rows x 32 fp32 columns
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool make_tmap_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) return false;
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols) * 2};
  cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static unsigned long long* g_tl = nullptr;
static int g_tl_cta = 0;
unsigned long long* timeline_buffer() { return g_tl; }
int timeline_cta() { return g_tl_cta; }

bool fill_postable(PosTable* t, int rows, int chunk, const int32_t* starts, int n) {
  std::memset(t, 0, sizeof(*t));
  if (chunk <= 0) {  // contiguous [0, rows)
    t->chunk = rows;
    t->nchunks = 1;
    t->start[0] = 0;
    t->tpc_shift = tpc_shift_of(rows);
    return true;
  }
  if (chunk % WF_TILE || n <= 0 || n > WF_MAX_CHUNKS || static_cast<int64_t>(n) * chunk != rows) return false;
  t->chunk = chunk;
  t->nchunks = n;
  t->tpc_shift = tpc_shift_of(chunk);
  for (int i = 0; i < n; ++i) t->start[i] = starts[i];
  return true;
}

}  // namespace wf

using namespace wf;

static thread_local char g_err[512];
const char* wf_static_error() { return g_err; }
static wf_status set_err(wf_status s, const char* msg) {
  std::snprintf(g_err, sizeof(g_err), "%s", msg);
  wf_clear_ctxless_error();
  return s;
}
wf_status wf_set_static_error(wf_status s, const char* msg) { return set_err(s, msg); }

// Debug aid: enable (cta >= 0) / disable (cta < 0) the block-kernel timeline of CTA
// (cta, head 0); wf_debug_timeline_read copies n words (after a device synchronize).
extern "C" wf_status wf_debug_timeline(int cta) {
  if (cta < 0) {
    g_tl = nullptr;
    return WF_OK;
  }
  static unsigned long long* buf = nullptr;
  const size_t bytes = size_t(4) * WF_TL_TILES * 8 * sizeof(unsigned long long);
  if (!buf && cudaMalloc(&buf, bytes) != cudaSuccess) return set_err(WF_ERR_CUDA, "timeline alloc");
  cudaMemset(buf, 0, bytes);
  g_tl = buf;
  g_tl_cta = cta;
  return WF_OK;
}
extern "C" wf_status wf_debug_timeline_read(unsigned long long* out, size_t n) {
  if (!g_tl) return set_err(WF_ERR_ARG, "timeline off");
  if (cudaDeviceSynchronize() != cudaSuccess) return set_err(WF_ERR_CUDA, "sync");
  const size_t cap = size_t(4) * WF_TL_TILES * 8;
  if (cudaMemcpy(out, g_tl, (n < cap ? n : cap) * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_err(WF_ERR_CUDA, "timeline copy");
  return WF_OK;
}

extern "C" wf_status wf_block_fwd(const void* q, const void* k, const void* v, int nq, int nk, int heads,
                                  int head_dim, int causal, int chunk, const int32_t* qstart, int nqchunks,
                                  const int32_t* kstart, int nkchunks, const float* o_in, const float* lse_in,
                                  float* o_out, void* o_bf16, float* lse_out, void* stream) {
  if (!q || !k || !v || !lse_out || (!o_out && !o_bf16)) return set_err(WF_ERR_ARG, "wf_block_fwd: null pointer");
  if ((o_in == nullptr) != (lse_in == nullptr)) return set_err(WF_ERR_ARG, "wf_block_fwd: o_in/lse_in must pair");
  if (nq <= 0 || nq % WF_TILE || nk < 0 || nk % WF_TILE) return set_err(WF_ERR_CONFIG, "wf_block_fwd: nq, nk must be multiples of 128");
  if (head_dim != 64 && head_dim != 72 && head_dim != 128) return set_err(WF_ERR_CONFIG, "wf_block_fwd: head_dim not in {64,72,128}");
  FwdArgs a{};
  a.nq = nq;
  a.nk = nk;
  a.heads = heads;
  a.causal = causal;
  if (causal) {
    if (!fill_postable(&a.qpos, nq, chunk, qstart, nqchunks) || !fill_postable(&a.kpos, nk, chunk, kstart, nkchunks))
      return set_err(WF_ERR_CONFIG, "wf_block_fwd: bad chunk table");
  } else {  // positions are irrelevant without a mask; contiguous tables drive the tile loops
    fill_postable(&a.qpos, nq, 0, nullptr, 0);
    fill_postable(&a.kpos, nk, 0, nullptr, 0);
  }
  a.scale_log2 = 1.4426950408889634f / std::sqrt(static_cast<float>(head_dim));
  a.o_in = o_in;
  a.lse_in = lse_in;
  a.o_out_f32 = o_out;
  a.o_out_bf16 = static_cast<__nv_bfloat16*>(o_bf16);
  a.lse_out = lse_out;
  a.lse_blk = nq;
  CUtensorMap tq, tk, tv;
  if (!make_tmap_rows(&tq, q, nq, heads, head_dim) || !make_tmap_rows(&tk, k, nk > 0 ? nk : WF_TILE, heads, head_dim) ||
      !make_tmap_rows(&tv, v, nk > 0 ? nk : WF_TILE, heads, head_dim))
    return set_err(WF_ERR_ARG, "wf_block_fwd: TMA map encode failed (alignment?)");
  cudaError_t e = launch_block_fwd(tq, tk, tv, a, head_dim, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_err(WF_ERR_CUDA, cudaGetErrorString(e));
  return WF_OK;
}

extern "C" wf_status wf_block_bwd(const void* q, const void* k, const void* v, const void* dO, const float* lse,
                                  const float* dsum, int nq, int nk, int heads, int head_dim, int causal, int chunk,
                                  const int32_t* qstart, int nqchunks, const int32_t* kstart, int nkchunks,
                                  float* dq_acc, float* dk_acc, float* dv_acc, int accumulate, void* stream) {
  if (!q || !k || !v || !dO || !lse || !dsum || !dq_acc || !dk_acc || !dv_acc)
    return set_err(WF_ERR_ARG, "wf_block_bwd: null pointer");
  if (nq < 0 || nq % WF_TILE || nk <= 0 || nk % WF_TILE) return set_err(WF_ERR_CONFIG, "wf_block_bwd: nq, nk must be multiples of 128");
  if (head_dim != 64 && head_dim != 72 && head_dim != 128) return set_err(WF_ERR_CONFIG, "wf_block_bwd: head_dim not in {64,72,128}");
  BwdArgs a{};
  a.nq = nq;
  a.nk = nk;
  a.heads = heads;
  a.causal = causal;
  if (causal) {
    if (!fill_postable(&a.qpos, nq, chunk, qstart, nqchunks) || !fill_postable(&a.kpos, nk, chunk, kstart, nkchunks))
      return set_err(WF_ERR_CONFIG, "wf_block_bwd: bad chunk table");
  } else {  // positions are irrelevant without a mask; contiguous tables drive the tile loops
    fill_postable(&a.qpos, nq, 0, nullptr, 0);
    fill_postable(&a.kpos, nk, 0, nullptr, 0);
  }
  a.scale = 1.f / std::sqrt(static_cast<float>(head_dim));
  a.scale_log2 = 1.4426950408889634f * a.scale;
  // the kernel takes -LSE log2(e) and -D / sqrt(d) (the runtime stores them that way once
  // per call); convert the caller's natural-log LSE and D into stream-ordered scratch
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t ns = static_cast<int64_t>(heads) * nq;
  float* conv = nullptr;
  if (ns > 0) {
    if (cudaMallocAsync(reinterpret_cast<void**>(&conv), 2 * ns * sizeof(float), st) != cudaSuccess)
      return set_err(WF_ERR_CUDA, "wf_block_bwd: scratch allocation failed");
    cudaError_t ce = launch_stats_convert(lse, dsum, conv, conv + ns, ns, a.scale, st);
    if (ce != cudaSuccess) return set_err(WF_ERR_CUDA, cudaGetErrorString(ce));
  }
  a.lse = conv;
  a.dsum = conv ? conv + ns : nullptr;
  a.dq_acc = dq_acc;
  a.dk_acc = dk_acc;
  a.dv_acc = dv_acc;
  a.dkv_accumulate = accumulate;
  a.stat_blk = nq > 0 ? nq : WF_TILE;
  CUtensorMap tq, tk, tv, tdo;
  if (!make_tmap_rows(&tq, q, nq > 0 ? nq : WF_TILE, heads, head_dim) || !make_tmap_rows(&tk, k, nk, heads, head_dim) ||
      !make_tmap_rows(&tv, v, nk, heads, head_dim) || !make_tmap_rows(&tdo, dO, nq > 0 ? nq : WF_TILE, heads, head_dim)) {
    if (conv) cudaFreeAsync(conv, st);
    return set_err(WF_ERR_ARG, "wf_block_bwd: TMA map encode failed (alignment?)");
  }
  cudaError_t e = launch_block_bwd(tq, tk, tv, tdo, a, head_dim, st);
  if (conv) cudaFreeAsync(conv, st);
  if (e != cudaSuccess) return set_err(WF_ERR_CUDA, cudaGetErrorString(e));
  return WF_OK;
}

extern "C" wf_status wf_gemm_bf16_t(const void* A, int a_mn, const void* B, int b_mn, int M, int N, int K, void* Y,
                                    void* stream) {
  if (!A || !B || !Y) return set_err(WF_ERR_ARG, "wf_gemm_bf16: null pointer");
  if ((reinterpret_cast<uintptr_t>(A) | reinterpret_cast<uintptr_t>(B) | reinterpret_cast<uintptr_t>(Y)) & 15)
    return set_err(WF_ERR_ARG, "wf_gemm_bf16: pointers must be 16-byte aligned");
  if (M <= 0 || M % 128 || N <= 0 || N % 128 || K <= 0 || K % 64)
    return set_err(WF_ERR_CONFIG, "wf_gemm_bf16: M, N multiples of 128 and K of 64 required");
  const int bn = N % 256 == 0 ? 256 : 128;
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.K = K;
  g.split = N;
  g.ndst[0] = 1;
  g.ld = N;
  g.out[0][0] = static_cast<__nv_bfloat16*>(Y);
  const bool pair = gemm_pair_ok(g, a_mn, b_mn);
  CUtensorMap ta, tb;
  const bool oka = a_mn ? make_tmap_2d(&ta, A, K, M, 64) : make_tmap_2d(&ta, A, M, K, 128);
  const bool okb = b_mn ? make_tmap_2d(&tb, B, K, N, 64) : make_tmap_2d(&tb, B, N, K, pair ? 128 : bn);
  if (!oka || !okb) return set_err(WF_ERR_ARG, "wf_gemm_bf16: TMA map encode failed");
  cudaError_t e = pair ? launch_gemm_pair(ta, tb, g, a_mn ? 1 : 0, b_mn ? 1 : 0, static_cast<cudaStream_t>(stream))
                       : launch_gemm_t(ta, tb, g, bn, a_mn ? 1 : 0, b_mn ? 1 : 0, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_err(WF_ERR_CUDA, cudaGetErrorString(e));
  return WF_OK;
}

extern "C" wf_status wf_gemm_bf16(const void* A, const void* B, int M, int N, int K, void* Y, void* stream) {
  return wf_gemm_bf16_t(A, 0, B, 0, M, N, K, Y, stream);
}
