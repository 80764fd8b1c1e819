// attn_fwd3.cu -- the block forward (PAPER.md:183 forward_iteration) with split softmax rows.
//
// Same contract and pipeline as wf_block_fwd_kernel (attn_fwd.cu: two 128-row query tiles
// per CTA, TMEM S_0 S_1 O_0 O_1, P written back over S as the TS operand of P V), head_dim
// 128, but every query row is handled by two softmax threads, each owning 64 of the 128
// key columns of a tile: 16 softmax warps (tile t, half hh, lane quadrant wq = warp % 4)
// plus a TMA and an MMA warp.  Per tile a thread loads 64 logits, the two halves exchange
// their partial row maxima through shared memory (a 64-thread named barrier per quadrant),
// and each half computes and stores its 64 probabilities and rescales its 64 output
// columns; the row sums stay partial until the epilogue.  Twice the warps share the
// exponential work of a tile, so the softmax phase that bounds the single-row kernel's
// period shortens and overlaps better with the MMAs.
#include <cstdlib>
#include <type_traits>

#include "common.h"
#include "sm100.cuh"

namespace wf {
using namespace sm100;

namespace {

#ifndef WF_FWD3_POLY
#define WF_FWD3_POLY 0  // every k-th exponential pair on the FMA pipe (0 = all on MUFU)
#endif
constexpr float kL2e = 1.4426950408889634f;
constexpr float kLn2c = 0.6931471805599453f;

struct Fwd3Cfg {
  static constexpr int D = 128;
  static constexpr int PANEL = 128 * 128;
  static constexpr int TILE = 2 * PANEL;
  static constexpr int OFF_Q = 0;                 // 2 query tiles
  static constexpr int OFF_K = 2 * TILE;          // 3 stages
  static constexpr int OFF_V = 5 * TILE;          // 2 stages
  static constexpr int OFF_X = 7 * TILE;          // partial maxima: [2 tiles][2 halves][128 rows] fp32
  static constexpr int OFF_BAR = OFF_X + 2048;
  static constexpr int SMEM = OFF_BAR + 256;
  static_assert(SMEM <= 232448, "shared memory budget");
};
enum { X_Q = 0, X_K = 1, X_KE = 4, X_V = 7, X_VE = 9, X_S = 11, X_P = 13, X_OF = 15, X_NUM = 17 };
constexpr int kX3Stages = 3;
constexpr int kTmaWarp = 16, kMmaWarp = 17;
constexpr int kF3Threads = 18 * 32;

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __launch_bounds__(kF3Threads, 1)
    wf_block_fwd3_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ FwdArgs a) {
  using Cfg = Fwd3Cfg;
  constexpr int D = Cfg::D;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + X_NUM * 8);
  float* xch = reinterpret_cast<float*>(smem + Cfg::OFF_X);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nqt = a.nq / WF_TILE;
  const int npairs = (nqt + 1) >> 1;
  const int pair = a.causal ? (npairs - 1 - blockIdx.x) : blockIdx.x;
  const int head = blockIdx.y;
  const int q0 = pair * 2 * WF_TILE;
  const bool hasB = q0 + WF_TILE < a.nq;
  const int ntile = hasB ? 2 : 1;
  const int qposA = a.causal ? tile_gpos(a.qpos, q0 / WF_TILE) : q0;
  const int qposB = (a.causal && hasB) ? tile_gpos(a.qpos, q0 / WF_TILE + 1) : q0 + WF_TILE;
  const bool has_state = a.o_in != nullptr;
  auto kind_of = [&](int t, int kp) -> int {
    if (t == 1 && !hasB) return 0;
    if (!a.causal) return 1;
    const int qp = t == 0 ? qposA : qposB;
    return kp > qp ? 0 : (kp == qp ? 2 : 1);
  };
  const int qbound = hasB ? max(qposA, qposB) : qposA;
  auto kv_iter = [&]() { return VisIter<true>(a.kpos, a.causal != 0, qbound); };

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    mbar_init(&bar[X_Q], 1);
    for (int i = 0; i < kX3Stages; ++i) {
      mbar_init(&bar[X_K + i], 1);
      mbar_init(&bar[X_KE + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[X_V + i], 1);
      mbar_init(&bar[X_VE + i], 1);
      mbar_init(&bar[X_S + i], 1);
      mbar_init(&bar[X_P + i], 256);  // both halves of the tile's 128 rows
      mbar_init(&bar[X_OF + i], 1);
    }
    fence_barrier_init();
  }
  if (warp == kMmaWarp) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == kTmaWarp) {
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      mbar_arrive_expect_tx(&bar[X_Q], ntile * Cfg::TILE);
      for (int t = 0; t < ntile; ++t)
        for (int p = 0; p < 2; ++p)
          tma_load_3d(smem + Cfg::OFF_Q + t * Cfg::TILE + p * Cfg::PANEL, &tmQ, &bar[X_Q], p * 64, head,
                      q0 + t * WF_TILE);
      int jj = 0, jt, kp;
      for (auto it = kv_iter(); it.next(a.kpos, jt, kp);) {
        const int st = jj % kX3Stages;
        if (jj >= kX3Stages) mbar_wait(&bar[X_KE + st], ((jj - kX3Stages) / kX3Stages) & 1);
        uint8_t* sk = smem + Cfg::OFF_K + st * Cfg::TILE;
        mbar_arrive_expect_tx(&bar[X_K + st], Cfg::TILE);
        for (int p = 0; p < 2; ++p) tma_load_3d(sk + p * Cfg::PANEL, &tmK, &bar[X_K + st], p * 64, head, jt * WF_TILE);
        ++jj;
      }
    } else if (lane == 1) {
      tma_prefetch_desc(&tmV);
      int jj = 0, jt, kp;
      for (auto it = kv_iter(); it.next(a.kpos, jt, kp);) {
        const int st = jj & 1;
        if (jj >= 2) mbar_wait(&bar[X_VE + st], ((jj - 2) >> 1) & 1);
        uint8_t* sv = smem + Cfg::OFF_V + st * Cfg::TILE;
        mbar_arrive_expect_tx(&bar[X_V + st], Cfg::TILE);
        for (int p = 0; p < 2; ++p) tma_load_3d(sv + p * Cfg::PANEL, &tmV, &bar[X_V + st], p * 64, head, jt * WF_TILE);
        ++jj;
      }
    }
  } else if (warp == kMmaWarp) {
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, 0, 0);
      constexpr uint32_t idO = idesc_bf16_f32(128, D, 0, 1);
      auto issue_s = [&](int t, int j) {
        const int st = j % kX3Stages;
        const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + t * Cfg::TILE);
        const uint32_t sK = smem_u32(smem + Cfg::OFF_K + st * Cfg::TILE);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const int p = k >> 2, kk = k & 3;
          mma_ss(tbase + t * 128, smem_desc_sw128(sQ + p * Cfg::PANEL + kk * 32, 16, 1024),
                 smem_desc_sw128(sK + p * Cfg::PANEL + kk * 32, 16, 1024), idS, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar[X_S + t]);
      };
      auto issue_pv = [&](int t, int j) {
        const int st = j & 1;
        mbar_wait(&bar[X_P + t], j & 1);
        if (t == 0) mbar_wait(&bar[X_V + st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + Cfg::OFF_V + st * Cfg::TILE);
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ts(tbase + 256 + t * 128, tbase + t * 128 + (k >> 2) * 64 + (k & 3) * 8,
                 smem_desc_sw128(sV + k * 2048, Cfg::PANEL, 1024), idO, (j > 0 || has_state || k > 0) ? 1u : 0u);
      };
      const int nvis = kv_iter().count(a.kpos);
      mbar_wait(&bar[X_Q], 0);
      for (int j = 0; j < nvis; ++j) {
        for (int t = 0; t < ntile; ++t) {
          if (j > 0) issue_pv(t, j - 1);
          if (t == 0) {
            mbar_wait(&bar[X_K + j % kX3Stages], (j / kX3Stages) & 1);
            tc_fence_after();
          }
          issue_s(t, j);
        }
        if (j > 0) mma_commit(&bar[X_VE + ((j - 1) & 1)]);
        mma_commit(&bar[X_KE + j % kX3Stages]);
      }
      if (nvis > 0) {
        for (int t = 0; t < ntile; ++t) {
          issue_pv(t, nvis - 1);
          mma_commit(&bar[X_OF + t]);
        }
        mma_commit(&bar[X_VE + ((nvis - 1) & 1)]);
      } else {
        for (int t = 0; t < ntile; ++t) mma_commit(&bar[X_OF + t]);
      }
    }
  } else if (warp < 16) {
    // ------------------------------------------------------------ softmax + epilogue
    const int t = warp >> 3, hh = (warp >> 2) & 1, wq = warp & 3;
    const int row = wq * 32 + lane;
    if (!(t == 1 && !hasB)) {
      const uint32_t tl = tbase + (static_cast<uint32_t>(wq * 32) << 16);
      const uint32_t cS = t * 128 + hh * 64;      // this half's 64 logits
      const uint32_t cP = t * 128 + hh * 64;      // its 64 probabilities, packed, over its own logits
      const uint32_t cO = 256 + t * 128 + hh * 64;
      const int grow = q0 + t * WF_TILE + row;
      const size_t orow = (static_cast<size_t>(grow) * a.heads + head) * D + hh * 64;
      float* xmine = xch + (t * 2 + hh) * 128 + row;
      const float* xpeer = xch + (t * 2 + (hh ^ 1)) * 128 + row;
      const int barid = 1 + t * 4 + wq;           // the two warps of this (tile, quadrant)
      float m = -INFINITY, l = 0.f;               // l: this half's partial row sum
      if (has_state) {
        const float ls = a.lse_in[stat_index(head, grow, a.heads, a.lse_blk)];
        m = ls * kL2e;
        l = (hh == 0 && ls != -INFINITY) ? 1.f : 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t r[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(a.o_in[orow + c * 16 + i]);
          tmem_st16(tl + cO + c * 16, r);
        }
        tmem_wait_st();
      }
      int j = 0;
      auto tile = [&](auto diag_c, const int kind) {
        constexpr bool DIAG = decltype(diag_c)::value;
        mbar_wait(&bar[X_S + t], j & 1);
        tc_fence_after();
        // pass 1: the partial row max over this half's 64 logits (two 32-column loads)
        float mxs[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld32(tl + cS + c * 32, r);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            float x = __uint_as_float(r[i]);
            if constexpr (DIAG) x = (kind == 0 || hh * 64 + c * 32 + i > row) ? -INFINITY : x;
            mxs[i & 3] = fmaxf(mxs[i & 3], x);
          }
        }
        const float mpart = fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3]));
        // exchange the partial maxima with the other half of the row
        *xmine = mpart;
        named_sync(barid, 64);
        const float mx = fmaxf(mpart, *xpeer);
        const float mcand = mx * a.scale_log2;
        const bool need = mcand > m + 8.0f;
        if (__any_sync(0xffffffffu, need)) {
          const float mnew = fmaxf(m, mcand);
          const float alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mnew);
          if (j > 0 || has_state) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              uint32_t r[16];
              tmem_ld16(tl + cO + c * 16, r);
              tmem_wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
              tmem_st16(tl + cO + c * 16, r);
            }
          }
          l *= alpha;
          m = mnew;
        }
        const float mm = (m == -INFINITY) ? 0.f : m;
        const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nm2 = make_float2(-mm, -mm);
        float2 rs2[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        // pass 2: 32 logits at a time -> probabilities, packed over the consumed logits
        // (chunk c's P lands in columns [16 c, 16 c + 16) of this half, logits already read)
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t r[32];
          tmem_ld32(tl + cS + c * 32, r);
          tmem_wait_ld();
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float x0 = __uint_as_float(r[2 * i]), x1 = __uint_as_float(r[2 * i + 1]);
            if constexpr (DIAG) {
              const int key = hh * 64 + c * 32 + 2 * i;
              if (kind == 0 || key > row) x0 = -INFINITY;
              if (kind == 0 || key + 1 > row) x1 = -INFINITY;
            }
            const float2 x = ffma2(make_float2(x0, x1), sc2, nm2);
#if WF_FWD3_POLY > 0
            const bool poly = !DIAG && ((c * 16 + i) % WF_FWD3_POLY) == WF_FWD3_POLY - 1;
            const float2 p = poly ? poly_exp2x2(x) : make_float2(fast_exp2(x.x), fast_exp2(x.y));
#else
            const float2 p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
#endif
            rs2[c] = fadd2(rs2[c], p);
            pk[i] = pack_bf16x2(p.x, p.y);
          }
          tmem_st16(tl + cP + c * 16, pk);
        }
        const float2 rsa = fadd2(rs2[0], rs2[1]);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bar[X_P + t]);
        l += rsa.x + rsa.y;
        ++j;
      };
      int jt, kp;
      for (auto it = kv_iter(); it.next(a.kpos, jt, kp);) {
        const int kind = kind_of(t, kp);
        if (kind == 1)
          tile(std::integral_constant<bool, false>{}, kind);
        else
          tile(std::integral_constant<bool, true>{}, kind);
      }
      // epilogue: combine the two partial row sums (the last exchange slot is free: the
      // peer read it before its last P arrival, which precedes the final O commit)
      mbar_wait(&bar[X_OF + t], 0);
      tc_fence_after();
      *xmine = l;
      named_sync(barid, 64);
      const float lt = l + *xpeer;
      const bool have_o = j > 0 || has_state;
      const float inv = lt > 0.f ? 1.f / lt : 0.f;
      if (hh == 0)
        a.lse_out[stat_index(head, grow, a.heads, a.lse_blk)] = lt > 0.f ? (m + __log2f(lt)) * kLn2c : -INFINITY;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t r[16];
        if (have_o) {
          tmem_ld16(tl + cO + c * 16, r);
          tmem_wait_ld();
        }
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = have_o ? __uint_as_float(r[i]) * inv : 0.f;
        if (a.o_out_f32) {
          float4* dst = reinterpret_cast<float4*>(a.o_out_f32 + orow + c * 16);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
        if (a.o_out_bf16) {
          uint4* dst = reinterpret_cast<uint4*>(a.o_out_bf16 + orow + c * 16);
#pragma unroll
          for (int i = 0; i < 2; ++i)
            dst[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kMmaWarp) tmem_dealloc(tbase, 512);
}

}  // namespace

bool block_fwd_split_ok(const FwdArgs& a, int D) {
  const char* e = std::getenv("WF_FWD_SPLIT");
  return e && e[0] == '1' && D == 128 && a.nq > 0;
}

cudaError_t launch_block_fwd_split(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                                   const FwdArgs& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(wf_block_fwd3_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd3Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid((a.nq / WF_TILE + 1) / 2, a.heads);
  wf_block_fwd3_kernel<<<grid, kF3Threads, Fwd3Cfg::SMEM, s>>>(tq, tk, tv, a);
  return cudaGetLastError();
}

}  // namespace wf
