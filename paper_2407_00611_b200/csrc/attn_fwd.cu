// attn_fwd.cu -- per-ring-step block attention forward for sm_100a.
//
// One launch = PAPER.md:183 `forward_iteration(lse, O, q_team, k_current, v_current)`
// for every (query tile, head): S = Q K^T (tcgen05, fp32 in TMEM), online softmax
// in registers (one thread per query row, running max in the log2 domain), P
// written back to TMEM as bf16 and O += P V with P as the TMEM A operand.  The
// (O, lse) state of earlier ring steps is loaded into TMEM before the first
// P V, so the logaddexp merge of SPEC.md:55 costs nothing extra (DESIGN.md
// "block-fwd").  Causal masking uses global positions (reading c14): tiles are
// 128-aligned ranges, so a (q tile, k tile) pair is either fully visible, fully
// masked (skipped) or the diagonal.
//
// CTA = 12 warps and two 128-row query tiles: warp 0 TMA producer, warp 1 TMEM allocator +
// single-thread MMA issuer, warps 4-7 / 8-11 softmax + epilogue of tile 0 / tile 1
// (thread <-> TMEM lane <-> query row).  TMEM: S_0 [0,128), S_1 [128,256) (P_t written
// back over S_t as bf16), O_0 [256,256+DP), O_1 [384,384+DP).
#include "common.h"
#include "sm100.cuh"

#include <type_traits>

namespace wf {
using namespace sm100;

namespace {

constexpr float kLog2e = 1.4426950408889634f;
#ifndef WF_FWD_FASTMAX
#define WF_FWD_FASTMAX 1  // 1: skip the row-max pass while the running max stays valid (see tile())
#endif
// Every k-th exponential pair on the FMA pipe (0 = all on MUFU).  Measured with the fast
// path of tile() (profiles/r02_fwd_experiments.md): at head_dim 72 the forward is bound by
// the exponentials (MUFU) and 1/4 on the FMA pipe saves 4 % of its time; at head_dim 128 it
// costs 2 %.  WF_POLY_EVERY overrides the per-head-dim default for experiments.
template <int D>
__host__ __device__ constexpr int poly_every() {
#ifdef WF_POLY_EVERY
  return WF_POLY_EVERY;
#else
  return D < 128 ? 4 : 0;
#endif
}
constexpr float kLn2 = 0.6931471805599453f;

template <int D>
struct FwdCfg {
  static constexpr int DP = (D + 15) / 16 * 16;   // MMA-padded head dim
  static constexpr int NP = (D + 63) / 64;        // 64-column smem panels per tile
  static constexpr int PANEL = 128 * 128;         // bytes of one [128 rows x 64 bf16] panel
  static constexpr int TILE = NP * PANEL;
  static constexpr int OFF_Q = 0;                 // 2 query tiles
  static constexpr int OFF_K = 2 * TILE;          // 3 stages (released after the S MMAs)
  static constexpr int OFF_V = 5 * TILE;          // 2 stages (released after the P V MMAs)
  static constexpr int OFF_BAR = 7 * TILE;
  static constexpr int SMEM = OFF_BAR + 256;
  static_assert(SMEM <= 232448, "shared memory budget");
};

// barriers: Q, K[2], V[2], KV-empty[2], S-full[2 tiles], P-full[2 tiles] (stride 4: slots for
// a split publication of P -- measured slower, so one arrive per tile), O-final[2 tiles].
enum { B_Q = 0, B_K = 1, B_KE = 4, B_V = 7, B_VE = 9, B_S = 11, B_P = 13, B_OF = 21, B_NUM = 23 };
constexpr int kKStages = 3;

constexpr int kFwdThreads = 12 * 32;  // TMA, MMA, 2 spare, 2 x 4 softmax warps
constexpr int kRegCtl = 56, kRegSoftmax = 224;
#ifndef WF_FWD_REGSPLIT
#define WF_FWD_REGSPLIT 1
#endif  // 56 + 2 x 224 <= 512 registers per lane slot

// Two 128-row query tiles per CTA share every K/V tile (half the K/V smem traffic per
// FLOP).  The tensor pipe alternates between them -- PV_0(j-1), S_0(j), PV_1(j-1), S_1(j)
// -- so each softmax warpgroup works on its tile while the MMAs of the other run.
// Because S_t(j) is issued after PV_t(j-1), the S_t(j) commit also retires PV_t(j-1):
// the O rescale needs no extra barrier.
template <int D>
__global__ void __launch_bounds__(kFwdThreads, 1)
    wf_block_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ FwdArgs a) {
  using Cfg = FwdCfg<D>;
  constexpr int DP = Cfg::DP;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + B_NUM * 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nqt = a.nq / WF_TILE;
  const int npairs = (nqt + 1) >> 1;
  // heavy pairs first: with zigzag units the later half of each unit sees more keys
  const int pair = a.causal ? (npairs - 1 - blockIdx.x) : blockIdx.x;
  const int head = blockIdx.y;
  const int q0 = pair * 2 * WF_TILE;
  const bool hasB = q0 + WF_TILE < a.nq;
  const int ntile = hasB ? 2 : 1;
  const int qposA = a.causal ? tile_gpos(a.qpos, q0 / WF_TILE) : q0;
  const int qposB = (a.causal && hasB) ? tile_gpos(a.qpos, q0 / WF_TILE + 1) : q0 + WF_TILE;
  const bool has_state = a.o_in != nullptr;
  const bool tlon = a.tl && static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x) == a.tl_cta;
  // kind of (query tile t, key tile starting at global position kp): 0 masked, 1 full, 2 diagonal
  auto kind_of = [&](int t, int kp) -> int {
    if (t == 1 && !hasB) return 0;
    if (!a.causal) return 1;
    const int qp = t == 0 ? qposA : qposB;
    return kp > qp ? 0 : (kp == qp ? 2 : 1);
  };
  // key tiles visible to either query tile: first position <= the larger query tile start
  const int qbound = hasB ? max(qposA, qposB) : qposA;
  auto kv_iter = [&]() { return VisIter<true>(a.kpos, a.causal != 0, qbound); };

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();  // SW128 operands need 1024-byte alignment
    mbar_init(&bar[B_Q], 1);
    for (int i = 0; i < kKStages; ++i) {
      mbar_init(&bar[B_K + i], 1);
      mbar_init(&bar[B_KE + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[B_V + i], 1);
      mbar_init(&bar[B_VE + i], 1);
      mbar_init(&bar[B_S + i], 1);
      for (int c = 0; c < 4; ++c) mbar_init(&bar[B_P + 4 * i + c], 128);
      mbar_init(&bar[B_OF + i], 1);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;
  // register split per SM sub-partition (one warp of each warpgroup shares it): the TMA /
  // MMA warpgroup keeps kRegCtl, the two softmax warpgroups take the rest (kRegSoftmax), so
  // a softmax thread holds its 128-column S row without spilling
  if (warp < 4) {
#if WF_FWD_REGSPLIT
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kRegCtl));
#endif
  if (warp == 0) {
    // ------------------------------------------------------------ TMA producers
    // lane 0: Q and the K ring (3 stages, freed by the S MMAs); lane 1: the V ring
    // (2 stages, freed by the P V MMAs).  Separate lanes keep a K load from queueing
    // behind a V stage that is still being read.
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      mbar_arrive_expect_tx(&bar[B_Q], ntile * Cfg::TILE);
      for (int t = 0; t < ntile; ++t)
        for (int p = 0; p < Cfg::NP; ++p)
          tma_load_3d(smem + Cfg::OFF_Q + t * Cfg::TILE + p * Cfg::PANEL, &tmQ, &bar[B_Q], p * 64, head,
                      q0 + t * WF_TILE);
      int jj = 0, jt, kp;
      for (auto it = kv_iter(); it.next(a.kpos, jt, kp);) {
        const int st = jj % kKStages;
        if (jj >= kKStages) mbar_wait(&bar[B_KE + st], ((jj - kKStages) / kKStages) & 1);
        tl_stamp(a.tl, tlon, 3, jj, 0);
        uint8_t* sk = smem + Cfg::OFF_K + st * Cfg::TILE;
        mbar_arrive_expect_tx(&bar[B_K + st], Cfg::TILE);
        for (int p = 0; p < Cfg::NP; ++p) tma_load_3d(sk + p * Cfg::PANEL, &tmK, &bar[B_K + st], p * 64, head, jt * WF_TILE);
        if (tlon && jj == 0) {  // debug timeline: arrival of Q and of the first K tile
          mbar_wait(&bar[B_Q], 0);
          tl_stamp(a.tl, tlon, 3, 0, 1);
          mbar_wait(&bar[B_K], 0);
          tl_stamp(a.tl, tlon, 3, 0, 2);
        }
        ++jj;
      }
    } else if (lane == 1) {
      tma_prefetch_desc(&tmV);
      int jj = 0, jt, kp;
      for (auto it = kv_iter(); it.next(a.kpos, jt, kp);) {
        const int st = jj & 1;
        if (jj >= 2) mbar_wait(&bar[B_VE + st], ((jj - 2) >> 1) & 1);
        uint8_t* sv = smem + Cfg::OFF_V + st * Cfg::TILE;
        mbar_arrive_expect_tx(&bar[B_V + st], Cfg::TILE);
        for (int p = 0; p < Cfg::NP; ++p) tma_load_3d(sv + p * Cfg::PANEL, &tmV, &bar[B_V + st], p * 64, head, jt * WF_TILE);
        ++jj;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idS = idesc_bf16_f32(128, 128, 0, 0);  // Q (K-major) x K (K-major)
      constexpr uint32_t idO = idesc_bf16_f32(128, DP, 0, 1);   // P (TMEM) x V (MN-major)
      // descriptor low words (desc_lo), hoisted out of the issue loops
      const uint32_t kQ = desc_lo(smem_u32(smem + Cfg::OFF_Q), 16);
      const uint32_t kK = desc_lo(smem_u32(smem + Cfg::OFF_K), 16);
      const uint32_t kV = desc_lo(smem_u32(smem + Cfg::OFF_V), Cfg::PANEL);
      auto issue_s = [&](int t, int j) {
        const int st = j % kKStages;
        const uint32_t q = kQ + ((t * Cfg::TILE) >> 4), kt = kK + ((st * Cfg::TILE) >> 4);
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) {
          const uint32_t off = ((k >> 2) * Cfg::PANEL + (k & 3) * 32) >> 4;
          mma_ss_lo(tbase + t * 128, q + off, kt + off, idS, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar[B_S + t]);
      };
      auto issue_pv = [&](int t, int j) {
        const int st = j & 1;
        mbar_wait(&bar[B_P + 4 * t], j & 1);
        if (t == 0) mbar_wait(&bar[B_V + st], (j >> 1) & 1);
        tc_fence_after();
        const uint32_t vt = kV + ((st * Cfg::TILE) >> 4);
        const uint32_t acc0 = (j > 0 || has_state) ? 1u : 0u;
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ts_lo(tbase + 256 + t * 128, tbase + t * 128 + k * 8, vt + k * 128, idO, k > 0 ? 1u : acc0);
      };
      const int nvis = kv_iter().count(a.kpos);
      mbar_wait(&bar[B_Q], 0);
      for (int j = 0; j < nvis; ++j) {
        tl_stamp(a.tl, tlon, 0, j, 0);
        for (int t = 0; t < ntile; ++t) {
          if (j > 0) issue_pv(t, j - 1);
          tl_stamp(a.tl, tlon, 0, j, 1 + 2 * t);
          if (t == 0) {
            mbar_wait(&bar[B_K + j % kKStages], (j / kKStages) & 1);
            tc_fence_after();
          }
          issue_s(t, j);
          tl_stamp(a.tl, tlon, 0, j, 2 + 2 * t);
        }
        if (j > 0) mma_commit(&bar[B_VE + ((j - 1) & 1)]);
        mma_commit(&bar[B_KE + j % kKStages]);
      }
      if (nvis > 0) {
        for (int t = 0; t < ntile; ++t) {
          issue_pv(t, nvis - 1);
          mma_commit(&bar[B_OF + t]);
        }
        mma_commit(&bar[B_VE + ((nvis - 1) & 1)]);
      } else {
        for (int t = 0; t < ntile; ++t) mma_commit(&bar[B_OF + t]);
      }
    }
  }
  } else {
#if WF_FWD_REGSPLIT
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kRegSoftmax));
#endif
    // ------------------------------------------------------------ softmax + epilogue (tile t)
    const int t = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    if (t == 1 && !hasB) {
      // no second tile in this CTA
    } else {
      const uint32_t tl = tbase + (static_cast<uint32_t>(wq * 32) << 16);
      const uint32_t cS = t * 128, cO = 256 + t * 128;
      const int grow = q0 + t * WF_TILE + row;
      const size_t orow = (static_cast<size_t>(grow) * a.heads + head) * D;
      float m = -INFINITY, l = 0.f;
      if (has_state) {
        const float ls = a.lse_in[stat_index(head, grow, a.heads, a.lse_blk)];
        m = ls * kLog2e;
        l = (ls == -INFINITY) ? 0.f : 1.f;
#pragma unroll
        for (int c = 0; c < DP / 16; ++c) {
          uint32_t r[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = c * 16 + i;
            r[i] = __float_as_uint(col < D ? a.o_in[orow + col] : 0.f);
          }
          tmem_st16(tl + cO + c * 16, r);
        }
        tmem_wait_st();
      }
      int j = 0;
      // one key tile; DIAG selects the masked variant (diagonal or fully masked tile) so the
      // common, fully visible path carries no per-element select and no register shuffle
      auto tile = [&](auto diag_c, const int kind) {
        constexpr bool DIAG = decltype(diag_c)::value;
        mbar_wait(&bar[B_S + t], j & 1);
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
          tl_stamp(a.tl, tlon && lane == 0 && wq == 0, 1 + t, j, 2);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            s[i] = __uint_as_float(r0[i]);
            s[32 + i] = __uint_as_float(r1[i]);
            s[64 + i] = __uint_as_float(r2[i]);
            s[96 + i] = __uint_as_float(r3[i]);
          }
        }
        if constexpr (DIAG) {
          const int lim = kind == 0 ? -1 : row;  // keys c <= lim are visible
#pragma unroll
          for (int c = 0; c < 128; ++c) s[c] = c > lim ? -INFINITY : s[c];
        }
        // exponentials of the tile against the max mm (log2 domain) -> P (bf16) in TMEM over
        // S; returns this row's sum of P
        auto exps = [&](const float mm) -> float {
          const float2 sc2 = make_float2(a.scale_log2, a.scale_log2), nm2 = make_float2(-mm, -mm);
          float2 rs2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pk[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 x = ffma2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nm2);
              constexpr int PE = poly_every<D>();
              float2 p;
              if constexpr (PE > 0) {
                // masked (-inf) logits exist only on DIAG tiles: those stay on MUFU (exact 0)
                const bool poly = !DIAG && ((c * 16 + i) % PE) == PE - 1;
                p = poly ? poly_exp2x2(x) : make_float2(fast_exp2(x.x), fast_exp2(x.y));
              } else {
                p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
              }
              rs2[c] = fadd2(rs2[c], p);
              pk[i] = pack_bf16x2(p.x, p.y);
            }
            tmem_st16(tl + cS + c * 16, pk);
          }
          const float2 rsa = fadd2(fadd2(rs2[0], rs2[1]), fadd2(rs2[2], rs2[3]));
          return rsa.x + rsa.y;
        };
        // Fast path (no row-max pass): exponentials against the running max m.  P may then
        // exceed 1 -- harmless in bf16/fp32 as long as no logit is more than 2^6 above m in
        // the log2 domain, which the row sum reveals (p <= sum < 2^64).  Otherwise, and on a
        // row's first visible tile (m = -inf), the slow path takes the row max and applies
        // the lazy rescale (threshold 2^8) before redoing the exponentials.
        float rs = 0.f;
        bool slow = !WF_FWD_FASTMAX || __any_sync(0xffffffffu, m == -INFINITY);
        if (!slow) {
          rs = exps(m);
          slow = __any_sync(0xffffffffu, !(rs < 1.8446744e19f));  // 2^64, also inf / nan
        }
        if (slow) {
          // row max as 8 independent chains (3-input FMNMX), then a small tree: a single
          // 128-long dependent chain would cost ~500 cycles of latency per tile
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
          if (__any_sync(0xffffffffu, need)) {
            const float mnew = fmaxf(m, mcand);
            const float alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mnew);
            if (j > 0 || has_state) {
              // PV_t(j-1) retired with the S_t(j) commit (issued before it)
#pragma unroll
              for (int c = 0; c < DP / 16; ++c) {
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
          tl_stamp(a.tl, tlon && lane == 0 && wq == 0, 1 + t, j, 3);
          rs = exps((m == -INFINITY) ? 0.f : m);
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&bar[B_P + 4 * t]);
        tl_stamp(a.tl, tlon && lane == 0 && wq == 0, 1 + t, j, 1);
        l += rs;
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
      mbar_wait(&bar[B_OF + t], 0);
      tc_fence_after();
      const bool have_o = j > 0 || has_state;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      a.lse_out[stat_index(head, grow, a.heads, a.lse_blk)] = l > 0.f ? (m + __log2f(l)) * kLn2 : -INFINITY;
#pragma unroll
      for (int c = 0; c < DP / 16; ++c) {
        uint32_t r[16];
        if (have_o) {
          tmem_ld16(tl + cO + c * 16, r);
          tmem_wait_ld();
        }
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = have_o ? __uint_as_float(r[i]) * inv : 0.f;
        if (c * 16 + 16 <= D) {
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
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = c * 16 + i;
            if (col < D) {
              if (a.o_out_f32) a.o_out_f32[orow + col] = v[i];
              if (a.o_out_bf16) a.o_out_bf16[orow + col] = __float2bfloat16_rn(v[i]);
            }
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, 512);
}

template <int D>
cudaError_t launch_fwd_d(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const FwdArgs& a,
                         cudaStream_t s) {
  using Cfg = FwdCfg<D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(wf_block_fwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((a.nq / WF_TILE + 1) / 2, a.heads);
  FwdArgs b = a;
  b.tl = timeline_buffer();
  b.tl_cta = timeline_cta();
  wf_block_fwd_kernel<D><<<grid, kFwdThreads, Cfg::SMEM, s>>>(tq, tk, tv, b);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_block_fwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv, const FwdArgs& a,
                             int D, cudaStream_t s) {
  if (a.nq <= 0 || a.nq % WF_TILE || a.nk % WF_TILE) return cudaErrorInvalidValue;
  switch (D) {
    case 128: return launch_fwd_d<128>(tq, tk, tv, a, s);
    case 64: return launch_fwd_d<64>(tq, tk, tv, a, s);
    case 72: return launch_fwd_d<72>(tq, tk, tv, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace wf
