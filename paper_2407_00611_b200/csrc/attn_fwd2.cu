// attn_fwd2.cu -- the block forward (PAPER.md:183 forward_iteration) on CTA pairs.
//
// Same contract as wf_block_fwd_kernel (attn_fwd.cu); used for head_dim 128 when the query
// rows fill whole pairs of pairs (nq % 512 == 0).  A cluster of two CTAs owns four 128-row
// query tiles (two per CTA); the even CTA issues M = 256 `tcgen05.mma.cta_group::2` MMAs
// whose A rows come from both CTAs (Q for S, P for O += P V) and whose B operand is split
// between them: each CTA loads 64 of the 128 keys of a K tile and 64 of the 128 head dims
// of a V tile.  That halves the per-SM K/V traffic, and the shared memory it frees holds P
// (bf16) for both tiles, so P no longer overwrites S in TMEM: S_t(j+1) is issued as soon as
// softmax_t(j) has loaded S_t(j) into registers, and the MMAs of the next key tile overlap
// the softmax of this one instead of following it (the single-CTA kernel's per-tile chain
// S -> softmax -> P V -> S).
//
// Roles per CTA (12 warps): warp 0 lane 0 TMA for Q and the K ring, lane 1 the V ring;
// warp 1 TMEM allocator (both CTAs) + MMA issuer (even CTA only); warps 4-7 / 8-11 softmax
// + epilogue of tile 0 / tile 1 (thread = query row = TMEM lane).  TMEM: S_0 [0,128),
// S_1 [128,256), O_0 [256,384), O_1 [384,512).  Shared: Q 2 x 32 KB, K 3 x 16 KB,
// V 2 x 16 KB, P 2 x 32 KB.  Barriers live at the same offset in both CTAs; the even CTA's
// copies of K/V/Q-full, S-loaded and P-ready count both CTAs, its MMA commits are
// multicast to both.
#include <cstdlib>
#include <type_traits>

#include "common.h"
#include "sm100.cuh"

namespace wf {
using namespace sm100;

namespace {

#ifndef WF_FWD2_STAGGER
#define WF_FWD2_STAGGER 1
#endif
#ifndef WF_FWD2_POLY
#define WF_FWD2_POLY 0  // every k-th exponential pair on the FMA pipe (0 = all on MUFU)
#endif
constexpr float kLog2e2 = 1.4426950408889634f;
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
constexpr float kLn2b = 0.6931471805599453f;

struct Fwd2Cfg {
  static constexpr int QT = 32768;           // one 128 x 128 bf16 query tile (2 panels)
  static constexpr int KT = 16384;           // this CTA's 64 keys x 128 dims (2 panels of 8 KB)
  static constexpr int VT = 16384;           // this CTA's 64 dims of 128 keys (1 panel)
  static constexpr int PT = 32768;           // P of one tile: 128 rows x 128 keys bf16
  static constexpr int KST = 3, VST = 2;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = 2 * QT;
  static constexpr int OFF_V = OFF_K + KST * KT;
  static constexpr int OFF_P = OFF_V + VST * VT;
  static constexpr int OFF_BAR = OFF_P + 2 * PT;
  static constexpr int SMEM = OFF_BAR + 256;
  static_assert(SMEM <= 232448, "shared memory budget");
};
enum {
  F_Q = 0, F_K = 1, F_KE = 4, F_V = 7, F_VE = 9, F_S = 11, F_SL = 13, F_P = 15, F_PVD = 17, F_OF = 19, F_NUM = 21
};
constexpr int kF2Threads = 12 * 32;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kF2Threads, 1)
    wf_block_fwd2_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK64,
                         const __grid_constant__ CUtensorMap tmV, const __grid_constant__ FwdArgs a) {
  using Cfg = Fwd2Cfg;
  constexpr int D = 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + F_NUM * 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const int npairs = a.nq / (2 * WF_TILE);  // even (nq % 512 == 0)
  auto pair_of = [&](int bx) { return a.causal ? (npairs - 1 - bx) : bx; };
  const int pair = pair_of(blockIdx.x);
  const int peer_pair = pair_of(blockIdx.x ^ 1);
  const int head = blockIdx.y;
  const int q0 = pair * 2 * WF_TILE;
  auto tpos = [&](int pr, int t) { return a.causal ? tile_gpos(a.qpos, pr * 2 + t) : (pr * 2 + t) * WF_TILE; };
  const int qposA = tpos(pair, 0), qposB = tpos(pair, 1);
  const bool has_state = a.o_in != nullptr;
  const bool tlon = a.tl && static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x) == a.tl_cta;
  auto kind_of = [&](int t, int kp) -> int {
    if (!a.causal) return 1;
    const int qp = t == 0 ? qposA : qposB;
    return kp > qp ? 0 : (kp == qp ? 2 : 1);
  };
  // the pair shares every key tile: visible if visible to any of its four query tiles
  const int qbound = max(max(qposA, qposB), max(tpos(peer_pair, 0), tpos(peer_pair, 1)));
  auto kv_iter = [&]() { return VisIter<true>(a.kpos, a.causal != 0, qbound); };

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    mbar_init(&bar[F_Q], 1);
    for (int i = 0; i < Cfg::KST; ++i) {
      mbar_init(&bar[F_K + i], 1);
      mbar_init(&bar[F_KE + i], 2);  // both tiles' S MMAs
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[F_V + i], 1);
      mbar_init(&bar[F_VE + i], 2);
      mbar_init(&bar[F_S + i], 1);
      mbar_init(&bar[F_SL + i], 8);  // 4 warps x 2 CTAs
      mbar_init(&bar[F_P + i], 8);
      mbar_init(&bar[F_PVD + i], 1);
      mbar_init(&bar[F_OF + i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc2(tmem_slot, 512);
    tmem_relinquish2();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK64);
      if (cr == 0) mbar_arrive_expect_tx(&bar[F_Q], 2 * 2 * Cfg::QT);
      for (int t = 0; t < 2; ++t)
        for (int p = 0; p < 2; ++p)
          tma_load_3d_pair(smem + Cfg::OFF_Q + t * Cfg::QT + p * 16384, &tmQ, &bar[F_Q], p * 64, head,
                           q0 + t * WF_TILE);
      int jj = 0, jt, kp;
      for (auto it = kv_iter(); it.next(a.kpos, jt, kp);) {
        const int st = jj % Cfg::KST;
        if (jj >= Cfg::KST) mbar_wait(&bar[F_KE + st], ((jj - Cfg::KST) / Cfg::KST) & 1);
        uint8_t* sk = smem + Cfg::OFF_K + st * Cfg::KT;
        if (cr == 0) mbar_arrive_expect_tx(&bar[F_K + st], 2 * Cfg::KT);
        for (int p = 0; p < 2; ++p)
          tma_load_3d_pair(sk + p * 8192, &tmK64, &bar[F_K + st], p * 64, head, jt * WF_TILE + cr * 64);
        ++jj;
      }
    } else if (lane == 1) {
      tma_prefetch_desc(&tmV);
      int jj = 0, jt, kp;
      for (auto it = kv_iter(); it.next(a.kpos, jt, kp);) {
        const int st = jj & 1;
        if (jj >= 2) mbar_wait(&bar[F_VE + st], ((jj - 2) >> 1) & 1);
        uint8_t* sv = smem + Cfg::OFF_V + st * Cfg::VT;
        if (cr == 0) mbar_arrive_expect_tx(&bar[F_V + st], 2 * Cfg::VT);
        tma_load_3d_pair(sv, &tmV, &bar[F_V + st], cr * 64, head, jt * WF_TILE);
        ++jj;
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ------------------------------------------------------------ MMA issuers (even CTA)
    if (cr == 0 && lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(256, 128, 0, 0);  // Q x K^T, K split by keys
      constexpr uint32_t idO = idesc_bf16_f32(256, 128, 0, 1);  // P x V, V split by dims
      auto issue_s = [&](int t, int j) {
        const int st = j % Cfg::KST;
        const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + t * Cfg::QT);
        const uint32_t sK = smem_u32(smem + Cfg::OFF_K + st * Cfg::KT);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int p = k >> 2, kk = k & 3;
          mma2_ss(tbase + t * 128, smem_desc_sw128(sQ + p * 16384 + kk * 32, 16, 1024),
                  smem_desc_sw128(sK + p * 8192 + kk * 32, 16, 1024), idS, k > 0 ? 1u : 0u);
        }
        mma2_commit_mc(&bar[F_S + t], 0x3);
      };
      auto issue_pv = [&](int t, int j) {
        const int st = j & 1;
        const uint32_t sP = smem_u32(smem + Cfg::OFF_P + t * Cfg::PT);
        const uint32_t sV = smem_u32(smem + Cfg::OFF_V + st * Cfg::VT);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const int p = k >> 2, kk = k & 3;
          mma2_ss(tbase + 256 + t * 128, smem_desc_sw128(sP + p * 16384 + kk * 32, 16, 1024),
                  smem_desc_sw128(sV + k * 2048, 16384, 1024), idO, (j > 0 || has_state || k > 0) ? 1u : 0u);
        }
        mma2_commit_mc(&bar[F_PVD + t], 0x3);
      };
      // one issuing thread per query tile (warps 1 and 2): the two tiles' S / P V chains are
      // independent, so neither waits behind the other's softmax; K and V stages are
      // released by both (count 2)
      const int t = warp - 1;
      const int nvis = kv_iter().count(a.kpos);
      mbar_wait(&bar[F_Q], 0);
      if (nvis > 0) {
#if WF_FWD2_STAGGER
        // start tile 1 after tile 0's first softmax: the two softmax warpgroups then take
        // their MUFU-heavy exponential phases in alternation instead of at the same time
        if (t == 1) mbar_wait(&bar[F_P + 0], 0);
#endif
        mbar_wait(&bar[F_K], 0);
        tc_fence_after();
        issue_s(t, 0);
        mma2_commit_mc(&bar[F_KE], 0x3);
      }
      for (int j = 0; j < nvis; ++j) {
        if (j + 1 < nvis) {
          const int st = (j + 1) % Cfg::KST;
          mbar_wait(&bar[F_K + st], ((j + 1) / Cfg::KST) & 1);
          mbar_wait(&bar[F_SL + t], j & 1);  // softmax_t(j) holds S_t(j) in registers
          tc_fence_after();
          issue_s(t, j + 1);
          tl_stamp(a.tl, tlon, 0, j, t);
          mma2_commit_mc(&bar[F_KE + st], 0x3);
        }
        mbar_wait(&bar[F_V + (j & 1)], (j >> 1) & 1);
        mbar_wait(&bar[F_P + t], j & 1);
        tc_fence_after();
        issue_pv(t, j);
        tl_stamp(a.tl, tlon, 0, j, 2 + t);
        mma2_commit_mc(&bar[F_VE + (j & 1)], 0x3);
      }
      mma2_commit_mc(&bar[F_OF + t], 0x3);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax + epilogue (tile t)
    const int t = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t tl = tbase + (static_cast<uint32_t>(wq * 32) << 16);
    const uint32_t cS = t * 128, cO = 256 + t * 128;
    const int grow = q0 + t * WF_TILE + row;
    const size_t orow = (static_cast<size_t>(grow) * a.heads + head) * D;
    uint8_t* prow = smem + Cfg::OFF_P + t * Cfg::PT + (row >> 3) * 1024 + (row & 7) * 128;
    float m = -INFINITY, l = 0.f;
    if (has_state) {
      const float ls = a.lse_in[stat_index(head, grow, a.heads, a.lse_blk)];
      m = ls * kLog2e2;
      l = (ls == -INFINITY) ? 0.f : 1.f;
#pragma unroll
      for (int c = 0; c < D / 16; ++c) {
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
      mbar_wait(&bar[F_S + t], j & 1);
      tc_fence_after();
      tl_stamp(a.tl, tlon && lane == 0 && wq == 0, 1 + t, j, 0);
      float s[128];
      {
        uint32_t r0[32], r1[32], r2[32], r3[32];
        tmem_ld32(tl + cS + 0, r0);
        tmem_ld32(tl + cS + 32, r1);
        tmem_ld32(tl + cS + 64, r2);
        tmem_ld32(tl + cS + 96, r3);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = __uint_as_float(r0[i]);
          s[32 + i] = __uint_as_float(r1[i]);
          s[64 + i] = __uint_as_float(r2[i]);
          s[96 + i] = __uint_as_float(r3[i]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&bar[F_SL + t], 0);  // S_t may be overwritten
      tl_stamp(a.tl, tlon && lane == 0 && wq == 0, 1 + t, j, 1);
      if constexpr (DIAG) {
        const int lim = kind == 0 ? -1 : row;
#pragma unroll
        for (int c = 0; c < 128; ++c) s[c] = c > lim ? -INFINITY : s[c];
      }
      float mxs[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) mxs[k] = fmaxf(s[k], s[8 + k]);
#pragma unroll
      for (int c = 16; c < 128; c += 16)
#pragma unroll
        for (int k = 0; k < 8; ++k) mxs[k] = fmaxf(mxs[k], fmaxf(s[c + k], s[c + 8 + k]));
      const float mx = fmaxf(fmaxf(fmaxf(mxs[0], mxs[1]), fmaxf(mxs[2], mxs[3])),
                             fmaxf(fmaxf(mxs[4], mxs[5]), fmaxf(mxs[6], mxs[7])));
      const float mcand = mx * a.scale_log2;
      const bool need = mcand > m + 8.0f;
      bool pv_done = false;
      if (__any_sync(0xffffffffu, need)) {
        const float mnew = fmaxf(m, mcand);
        const float alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mnew);
        if (j > 0 || has_state) {
          if (j > 0) {  // O_t must include P_t(j-1) V before it is rescaled
            mbar_wait(&bar[F_PVD + t], (j - 1) & 1);
            tc_fence_after();
            pv_done = true;
          }
#pragma unroll
          for (int c = 0; c < D / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(tl + cO + c * 16, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st16(tl + cO + c * 16, r);
          }
          tmem_wait_st();
        }
        l *= alpha;
        m = mnew;
      }
      tl_stamp(a.tl, tlon && lane == 0 && wq == 0, 1 + t, j, 2);
      const float mm = (m == -INFINITY) ? 0.f : m;
      const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nm2 = make_float2(-mm, -mm);
      float2 rs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      // the P_t buffer is free once P_t(j-1) V has been consumed
      if (j > 0 && !pv_done) mbar_wait(&bar[F_PVD + t], (j - 1) & 1);
#pragma unroll
      for (int c = 0; c < 4; ++c) {  // 32 keys per chunk = 4 16-byte granules of one panel row
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 x = ffma2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nm2);
#if WF_FWD2_POLY > 0
          // a share of the exponentials on the FMA pipe: the softmax warps' MUFU work, not
          // the tensor pipe, sets this kernel's period (masked -inf logits stay on MUFU)
          const bool poly = !DIAG && ((c * 16 + i) % WF_FWD2_POLY) == WF_FWD2_POLY - 1;
          const float2 p = poly ? poly_exp2x2(x) : make_float2(fast_exp2(x.x), fast_exp2(x.y));
#else
          const float2 p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
#endif
          rs2[c] = fadd2(rs2[c], p);
          pk[i] = pack_bf16x2(p.x, p.y);
        }
        // keys [32c, 32c + 32): panel c >> 1, granules 4 (c & 1) .. 4 (c & 1) + 3
        uint8_t* pp = prow + (c >> 1) * 16384;
#pragma unroll
        for (int g4 = 0; g4 < 4; ++g4) {
          const int gi = (c & 1) * 4 + g4;
          *reinterpret_cast<uint4*>(pp + ((gi ^ (row & 7)) << 4)) =
              make_uint4(pk[4 * g4], pk[4 * g4 + 1], pk[4 * g4 + 2], pk[4 * g4 + 3]);
        }
      }
      const float2 rsa = fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3]));
      fence_proxy_async_smem();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&bar[F_P + t], 0);
      tl_stamp(a.tl, tlon && lane == 0 && wq == 0, 1 + t, j, 3);
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
    // epilogue
    mbar_wait(&bar[F_OF + t], 0);
    tc_fence_after();
    const bool have_o = j > 0 || has_state;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    a.lse_out[stat_index(head, grow, a.heads, a.lse_blk)] = l > 0.f ? (m + __log2f(l)) * kLn2b : -INFINITY;
#pragma unroll
    for (int c = 0; c < D / 16; ++c) {
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
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) tmem_dealloc2(tbase, 512);
}

}  // namespace

// Opt-in (WF_FWD_PAIR=1): measured equal to the single-CTA kernel (13.0-13.3 M vs 13.1 M
// cycles at GPT 32K) -- the softmax warps' exponential phase, not the MMA chain or the
// operand traffic, sets the period of both.  Kept, tested, as the CTA-pair groundwork.
bool block_fwd_pair_ok(const FwdArgs& a, int D) {
  const char* e = std::getenv("WF_FWD_PAIR");
  return e && e[0] == '1' && D == 128 && a.nq > 0 && a.nq % (4 * WF_TILE) == 0;
}

cudaError_t launch_block_fwd_pair(const CUtensorMap& tq, const CUtensorMap& tk64, const CUtensorMap& tv,
                                  const FwdArgs& a, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(wf_block_fwd2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, Fwd2Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  dim3 grid(a.nq / (2 * WF_TILE), a.heads);
  wf_block_fwd2_kernel<<<grid, kF2Threads, Fwd2Cfg::SMEM, s>>>(tq, tk64, tv, a);
  return cudaGetLastError();
}

}  // namespace wf
