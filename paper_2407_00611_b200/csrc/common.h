// common.h -- host/device shared definitions of the WallFacer B200 library.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define WF_MAX_CHUNKS 32
#define WF_TILE 128

namespace wf {

// Global-position table of a row buffer made of equal chunks (zigzag halves or
// whole units).  Row r of the buffer sits at global token
//   start[r / chunk] + r % chunk.
// chunk is a multiple of WF_TILE, so every 128-row tile is one contiguous range.
// Index of (head, row) in a per-row statistic stored as [rows/blk][heads][blk]
// (blk = rows gives the plain [heads, rows] layout; blk = one unit's rows gives the
// member-major layout of team-gathered statistics).
__host__ __device__ __forceinline__ int64_t stat_index(int head, int row, int heads, int blk) {
  return static_cast<int64_t>(row / blk) * heads * blk + static_cast<int64_t>(head) * blk + row % blk;
}

struct PosTable {
  int chunk;                      // rows per chunk (multiple of 128)
  int nchunks;
  int tpc_shift;                  // log2(chunk / 128) when that is a power of two, else -1
  int start[WF_MAX_CHUNKS];       // global start of each chunk
};

// Global position of the first row of 128-row tile `tile` (no integer division on the
// power-of-two fast path: it runs once per tile in every warp role).
__host__ __device__ __forceinline__ int tile_gpos(const PosTable& t, int tile) {
  if (t.tpc_shift >= 0) {
    const int c = tile >> t.tpc_shift;
    return t.start[c] + ((tile - (c << t.tpc_shift)) << 7);
  }
  const int row0 = tile * 128;
  return t.start[row0 / t.chunk] + row0 % t.chunk;
}
// Visible 128-row tiles of a block, chunk by chunk.  Positions increase inside a chunk, so
// under the causal rule the visible tiles of a chunk are a prefix (KEYS: first position
// <= bound, the query side's last tile start) or a suffix (QUERIES: first position >=
// bound, the key tile's start); one table read per chunk instead of a position lookup per
// tile (the per-tile lookups went through local memory and cost ~40k cycles per CTA).
template <bool KEYS>
struct VisIter {
  int c, i, hi, s, tpc, bound;
  bool causal;
  __device__ __forceinline__ VisIter(const PosTable& t, bool causal_, int bound_)
      : c(-1), i(0), hi(0), s(0), tpc(t.chunk >> 7), bound(bound_), causal(causal_) {}
  __device__ __forceinline__ void range(int st, int& lo, int& h) const {
    if (!causal) {
      lo = 0;
      h = tpc;
    } else if (KEYS) {
      const int d = bound - st;
      lo = 0;
      h = d < 0 ? 0 : ((d >> 7) + 1 < tpc ? (d >> 7) + 1 : tpc);
    } else {
      const int d = bound - st;
      lo = d <= 0 ? 0 : (((d + 127) >> 7) < tpc ? ((d + 127) >> 7) : tpc);
      h = tpc;
    }
  }
  // next visible tile: its index in the block and its first global position
  __device__ __forceinline__ bool next(const PosTable& t, int& tile, int& pos) {
    while (i >= hi) {
      if (++c >= t.nchunks) return false;
      s = t.start[c];
      range(s, i, hi);
    }
    tile = c * tpc + i;
    pos = s + (i << 7);
    ++i;
    return true;
  }
  __device__ __forceinline__ int count(const PosTable& t) const {
    int n = 0;
    for (int cc = 0; cc < t.nchunks; ++cc) {
      int lo, h;
      range(t.start[cc], lo, h);
      n += h - lo;
    }
    return n;
  }
};

inline int tpc_shift_of(int chunk) {
  const int tpc = chunk / 128;
  int sh = 0;
  while ((1 << sh) < tpc) ++sh;
  return (1 << sh) == tpc ? sh : -1;
}

// Arguments of one block-forward launch (PAPER.md:183 forward_iteration):
// the (O, lse) state of the query rows is merged with attention against one K/V block.
struct FwdArgs {
  int nq, nk, heads;
  int causal;
  PosTable qpos, kpos;
  float scale_log2;               // log2(e) / sqrt(head_dim)
  const float* o_in;              // optional state: fp32 [nq, heads, D] (normalised O)
  const float* lse_in;            // optional state: fp32 [heads, nq] natural log
  float* o_out_f32;               // state out (fp32) or null
  __nv_bfloat16* o_out_bf16;      // final out (bf16) or null
  float* lse_out;                 // [heads, nq]
  int lse_blk;                    // lse layout: rows in blocks of lse_blk, [nq/blk][heads][blk]
  unsigned long long* tl;         // debug timeline (null = off), see wf_debug_timeline
  int tl_cta;
};

// Arguments of one block-backward launch (flash-attention backward):
// the stationary K/V block accumulates dK/dV, the travelling query rows accumulate dQ.
struct BwdArgs {
  int nq, nk, heads;
  int causal;
  PosTable qpos, kpos;
  float scale_log2;               // log2(e) / sqrt(head_dim)
  float scale;                    // 1 / sqrt(head_dim)
  const float* lse;               // [heads, nq] -LSE log2(e) of the query rows (final forward LSE,
                                  // natural log, converted by launch_dsum / launch_stats_convert)
  const float* dsum;              // [heads, nq] -D / sqrt(d), D = rowsum(dO o O)
  float* dq_acc;                  // fp32 [nq, heads, D] accumulated with atomics
  float* dk_acc;                  // fp32 [nk, heads, D] (accumulate if dkv_accumulate)
  float* dv_acc;
  __nv_bfloat16* dk_out;          // if non-null: write bf16 dK (and dV) instead of fp32 acc
  __nv_bfloat16* dv_out;
  int dkv_accumulate;             // 1: dk_acc += ; 0: dk_acc =
  int stat_blk;                   // lse/dsum layout: [nq/blk][heads][blk]
  unsigned long long* tl;         // debug timeline (null = off)
  int tl_cta;
};

// Host: encode a 3-D TMA map over a [rows, heads, D] bf16 tensor, box {64, 1, 128}, SW128.
bool make_tmap_rows(CUtensorMap* map, const void* base, int64_t rows, int heads, int D);
// same with a {64, 1, box_rows} box
bool make_tmap_rows_box(CUtensorMap* map, const void* base, int64_t rows, int heads, int D, int box_rows);
// Debug timeline (bench/profiling aid): when enabled, one CTA of every block kernel records
// clock64() stamps at slot ((role * WF_TL_TILES + tile) * 8 + event).
#define WF_TL_TILES 1024
unsigned long long* timeline_buffer();  // null when disabled
int timeline_cta();
// Host: 3-D TMA map over a [rows, heads, D] fp32 tensor, box {32, 1, 32}, SW128 (dQ reduce-add).
bool make_tmap_f32_rows(CUtensorMap* map, const void* base, int64_t rows, int heads, int D);

// Host: 2-D TMA map over a row-major [rows, cols] bf16 matrix, box {64, box_rows}, SW128.
bool make_tmap_2d(CUtensorMap* map, const void* base, int64_t rows, int64_t cols, int box_rows);

// Y = A B^T (bf16 in, fp32 accumulate, bf16 out), A [M, K], B [N, K] row-major (the QKV
// projection of PAPER.md Alg. 1 l.1).  Output column c belongs to part c / split (Q, K, V)
// at column c % split of a row-major [M, split] matrix with leading dimension ld; every
// tile is stored to ndst destinations of its part (the caller's tensor and, fused, the
// team members' gathered buffers over peer memory).
#define WF_GEMM_MAX_DST 6
struct GemmArgs {
  int M, N, K;
  int split;
  int ndst[3];                    // destinations per part
  int64_t ld;
  __nv_bfloat16* out[3][WF_GEMM_MAX_DST];
};
cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int bn, cudaStream_t s);
// a_mn / b_mn: operand stored MN-major ([K, M] / [K, N]); its TMA map has 64 x 64 boxes.
cudaError_t launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int bn, int a_mn, int b_mn,
                          cudaStream_t s);
// CTA-pair (cta_group::2) variant for K-major A and B with M, N, split multiples of 256
// (used whenever it applies); its A and B maps both use 128-row boxes.
bool gemm_pair_ok(const GemmArgs& g, int a_mn, int b_mn);
// CTA-pair GEMM (256 x 256 tiles) for any operand layout; requires gemm_pair_ok
cudaError_t launch_gemm_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int a_mn, int b_mn,
                             cudaStream_t s);

cudaError_t launch_block_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const FwdArgs& a,
                             int D, cudaStream_t s);
cudaError_t launch_block_bwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                             const CUtensorMap& tdo, const BwdArgs& a, int D, cudaStream_t s);

}  // namespace wf

#define WF_MAX_PARTS 8
namespace wf {
// ReduceScatter_combine of the C partial (O, lse) states of this rank's rows.
struct MergeArgs {
  int rows, heads, D, nparts;
  const float* o[WF_MAX_PARTS];           // fp32 [rows, heads, D] each
  const float* lse[WF_MAX_PARTS];         // lse[j][head * lse_stride[j] + row]
  int64_t lse_stride[WF_MAX_PARTS];
  __nv_bfloat16* out;                     // [rows, heads, D]
  float* lse_out;                         // [heads, rows]
};
struct SumArgs {
  int64_t n;                              // elements (multiple of 4)
  int nparts;
  const float* parts[WF_MAX_PARTS];
  __nv_bfloat16* out;
};
cudaError_t launch_merge(const MergeArgs& a, cudaStream_t s);
cudaError_t launch_dsum(const __nv_bfloat16* dO, const __nv_bfloat16* O, const float* lse, float* nd, float* nl,
                        int rows, int heads, int D, float scale, cudaStream_t s);
// nl = -lse log2(e) (-inf kept), nd = -dsum scale, n elements
cudaError_t launch_stats_convert(const float* lse, const float* dsum, float* nl, float* nd, int64_t n, float scale,
                                 cudaStream_t s);
cudaError_t launch_sum(const SumArgs& a, cudaStream_t s);
}  // namespace wf

#define WF_MAX_SIG 64
namespace wf {
// A batch of flag updates (signal) or flag conditions (wait): dst[i] is a flag address,
// val[i] the count to publish / to wait for.
struct SigArgs {
  int n;
  uint32_t* dst[WF_MAX_SIG];
  uint32_t val[WF_MAX_SIG];
  // waits only: host-mapped failure words ([0] flag, [1] expected, [2] seen) written on a
  // timeout of timeout_ns; a wait that finds [0] set returns at once (fail fast)
  uint32_t* fail;
  uint64_t timeout_ns;
};
cudaError_t launch_signal_wait(const SigArgs& sig, const SigArgs& wait, cudaStream_t s);
}  // namespace wf
