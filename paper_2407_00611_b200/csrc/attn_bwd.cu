// attn_bwd.cu -- per-ring-step block attention backward for sm_100a.
//
// One launch = one step of WallFacer's backward inner loop: the
// K/V block is stationary (its dK/dV "maintained fixed on the corresponding GPU",
// PAPER.md:203) and the travelling query rows bring Q, dO, LSE and D = rowsum(dO o O);
// their dQ is accumulated and travels on.  The per-block math "mirrors ...
// flash-attention", written out in DESIGN.md:
//   S^T = K Q^T, P^T = exp(S^T/sqrt(d) - LSE), dV += P^T dO,
//   dP^T = V dO^T, dS^T = P^T o (dP^T - D), dK += dS^T Q / sqrt(d), dQ += dS K / sqrt(d).
//
// CTA per (128-row K/V tile, head); it loops over the visible 128-row query tiles.
// 14 warps: 0-3 dQ drain (TMEM -> smem -> bulk reduce-add into fp32 dQ, lane = query
// row), 4-11 compute (lane = key row, two warps per lane quadrant split the 128 query
// columns), 12 TMA producer, 13 TMEM allocator + MMA issuer.
// TMEM: S^T [0,128) (P^T bf16 over [0,64)), dV [128,128+DP), dP^T [256,384)
// (dS^T bf16 over [256,320), then dQ over [256,256+DP)), dK [384,384+DP).
#include "common.h"
#include "sm100.cuh"

namespace wf {
using namespace sm100;

namespace {


template <int D>
struct BwdCfg {
  static constexpr int DP = (D + 15) / 16 * 16;
  static constexpr int NP = (D + 63) / 64;
  static constexpr int PANEL = 128 * 128;
  static constexpr int TILE = NP * PANEL;
  static constexpr int QST = 2;                 // query-tile ring depth
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;        // QST stages
  static constexpr int OFF_DO = (2 + QST) * TILE;  // 1 stage
  static constexpr int OFF_DS = (3 + QST) * TILE;     // [128 kv] x [128 q] bf16 dS (2 SW128 panels)
  static constexpr int OFF_STG = OFF_DS + 2 * PANEL;  // dQ drain staging: per warp 2 x [32 rows][32 fp32]
  static constexpr int OFF_STAT = OFF_STG + 32768;    // 2 stages x (lse[128], dsum[128]) fp32
  static constexpr int OFF_BAR = OFF_STAT + 2 * 1024;
  static constexpr int SMEM = OFF_BAR + 192;
  static_assert(SMEM <= 232448, "shared memory budget");
};

enum {
  B_KV = 0, B_QF = 1, B_QE = 4, B_SF = 7, B_SE = 9, B_DOF = 11, B_DOE = 12, B_S = 13, B_DP = 14, B_P = 15,
  B_DS = 16, B_DQF = 17, B_DQE = 18, B_DSE = 19, B_DONE = 20, B_SL = 21, B_SRF = 22, B_NUM = 23
};

#ifndef WF_BWD_POLY_EVERY
#define WF_BWD_POLY_EVERY 0  // every k-th exponential pair of the P phase on the FMA pipe
#endif
constexpr int kThreads = 14 * 32;  // 4 dQ-drain + 8 compute + TMA + MMA warps
constexpr int kCompute = 256;

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// TMA tensor reduce-add of a [32 rows][32 fp32] SW128 smem box into global (fp32)
__device__ __forceinline__ void tma_reduce_add_3d(const CUtensorMap* map, const void* ssrc, int c0, int c1, int c2) {
  asm volatile("cp.reduce.async.bulk.tensor.3d.global.shared::cta.add.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(ssrc)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}
__device__ __forceinline__ void named_bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    wf_block_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                        const __grid_constant__ CUtensorMap tmDQ, const __grid_constant__ BwdArgs a) {
  using Cfg = BwdCfg<D>;
  constexpr int DP = Cfg::DP;
#ifndef WF_BWD_PARK
#define WF_BWD_PARK 1
#endif
  constexpr bool kPark = WF_BWD_PARK && DP > 64;  // park dQ's second half in free S^T columns
  constexpr int QST = Cfg::QST;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + B_NUM * 8);
  float* stat = reinterpret_cast<float*>(smem + Cfg::OFF_STAT);  // [stage][2][128]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int kt = blockIdx.x;
  const int head = blockIdx.y;
  const int k0 = kt * WF_TILE;
  const int kpos0 = a.causal ? tile_gpos(a.kpos, kt) : k0;
  // query tiles that see this key tile: first position >= kpos0 (kind 2 when equal)
  auto q_iter = [&]() { return VisIter<false>(a.qpos, a.causal != 0, kpos0); };
  auto kind_at = [&](int qp) -> int { return (a.causal && qp == kpos0) ? 2 : 1; };
  const bool tlon = a.tl && static_cast<int>(blockIdx.y * gridDim.x + blockIdx.x) == a.tl_cta;

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();  // SW128 operands need 1024-byte alignment
    mbar_init(&bar[B_KV], 1);
    for (int i = 0; i < QST; ++i) {
      mbar_init(&bar[B_QF + i], 1);
      mbar_init(&bar[B_QE + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[B_SF + i], 1);
      mbar_init(&bar[B_SE + i], kCompute);
    }
    mbar_init(&bar[B_DOF], 1);
    mbar_init(&bar[B_DOE], 1);
    mbar_init(&bar[B_S], 1);
    mbar_init(&bar[B_DP], 1);
    mbar_init(&bar[B_P], kCompute);
    mbar_init(&bar[B_DS], kCompute);
    mbar_init(&bar[B_DQF], 1);
    mbar_init(&bar[B_DQE], 128);
    mbar_init(&bar[B_DSE], 1);
    mbar_init(&bar[B_DONE], 1);
    mbar_init(&bar[B_SL], kCompute);
    mbar_init(&bar[B_SRF], 128);
    fence_barrier_init();
  }
  if (warp == 13) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 12) {
    // ------------------------------------------------------------ TMA producers
    // lane 0: K, V once, then the query ring (QST stages, freed by dK);
    // lane 1: the statistics ring (2 stages, freed by the compute warps) and dO (freed by dV).
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_arrive_expect_tx(&bar[B_KV], 2 * Cfg::TILE);
      for (int p = 0; p < Cfg::NP; ++p) {
        tma_load_3d(smem + Cfg::OFF_K + p * Cfg::PANEL, &tmK, &bar[B_KV], p * 64, head, k0);
        tma_load_3d(smem + Cfg::OFF_V + p * Cfg::PANEL, &tmV, &bar[B_KV], p * 64, head, k0);
      }
      int ii = 0;
      int it, qp;
      for (auto iq = q_iter(); iq.next(a.qpos, it, qp);) {
        const int st = ii % QST;
        if (ii >= QST) mbar_wait(&bar[B_QE + st], ((ii - QST) / QST) & 1);
        tl_stamp(a.tl, tlon, 3, ii, 0);
        mbar_arrive_expect_tx(&bar[B_QF + st], Cfg::TILE);
        for (int p = 0; p < Cfg::NP; ++p)
          tma_load_3d(smem + Cfg::OFF_Q + st * Cfg::TILE + p * Cfg::PANEL, &tmQ, &bar[B_QF + st], p * 64, head,
                      it * WF_TILE);
        ++ii;
      }
    } else if (lane == 1) {
      tma_prefetch_desc(&tmDO);
      int ii = 0;
      int it, qp;
      for (auto iq = q_iter(); iq.next(a.qpos, it, qp);) {
        const int ss = ii & 1;
        if (ii >= 2) mbar_wait(&bar[B_SE + ss], ((ii - 2) >> 1) & 1);
        mbar_arrive_expect_tx(&bar[B_SF + ss], 1024);
        const int64_t soff = stat_index(head, it * WF_TILE, a.heads, a.stat_blk);
        bulk_load(stat + ss * 256, a.lse + soff, 512, &bar[B_SF + ss]);
        bulk_load(stat + ss * 256 + 128, a.dsum + soff, 512, &bar[B_SF + ss]);
        if (ii >= 1) mbar_wait(&bar[B_DOE], (ii - 1) & 1);
        tl_stamp(a.tl, tlon, 3, ii, 1);
        mbar_arrive_expect_tx(&bar[B_DOF], Cfg::TILE);
        for (int p = 0; p < Cfg::NP; ++p)
          tma_load_3d(smem + Cfg::OFF_DO + p * Cfg::PANEL, &tmDO, &bar[B_DOF], p * 64, head, it * WF_TILE);
        ++ii;
      }
    }
  } else if (warp == 13) {
    // ------------------------------------------------------------ MMA issuer
    // Per query tile i: dP_i, [P_i] dV_i, S_{i+1}, [dS_i] dQ_i, dK_i.  S_{i+1} is issued as
    // soon as dV_i has consumed P_i from TMEM, so the compute warps' exp work of tile i+1
    // overlaps dQ_i / dK_i; dQ first so that its drain (which gates dP_{i+1}) starts early.
    if (lane == 0) {
      constexpr uint32_t idSP = idesc_bf16_f32(128, 128, 0, 0);   // K x Q^T, V x dO^T (both K-major)
      constexpr uint32_t idKV = idesc_bf16_f32(128, DP, 0, 1);    // P^T (TMEM) / dS^T (smem) x dO / Q (MN-major)
      constexpr uint32_t idQ = idesc_bf16_f32(128, DP, 1, 1);     // dS (smem, MN-major) x K (MN-major)
      // descriptor low words (desc_lo): K-major operands with LBO 16, MN-major with LBO = PANEL
      const uint32_t kK = desc_lo(smem_u32(smem + Cfg::OFF_K), 16);
      const uint32_t kKm = desc_lo(smem_u32(smem + Cfg::OFF_K), Cfg::PANEL);
      const uint32_t kV = desc_lo(smem_u32(smem + Cfg::OFF_V), 16);
      const uint32_t kDO = desc_lo(smem_u32(smem + Cfg::OFF_DO), 16);
      const uint32_t kDOm = desc_lo(smem_u32(smem + Cfg::OFF_DO), Cfg::PANEL);
      const uint32_t kDS = desc_lo(smem_u32(smem + Cfg::OFF_DS), 16);
      const uint32_t kDSm = desc_lo(smem_u32(smem + Cfg::OFF_DS), Cfg::PANEL);
      auto issue_s = [&](int i) {
        const int st = i % QST;
        const uint32_t kQ = desc_lo(smem_u32(smem + Cfg::OFF_Q + st * Cfg::TILE), 16);
        tl_stamp(a.tl, tlon, 0, i, 4);
        if (kPark && i >= 2) mbar_wait(&bar[B_SRF], (i - 2) & 1);  // drain of tile i-2 left S^T columns [64, 128)
        mbar_wait(&bar[B_QF + st], (i / QST) & 1);
        tl_stamp(a.tl, tlon, 0, i, 5);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) {
          const int p = k >> 2, kk = k & 3;
          const uint32_t off = (p * Cfg::PANEL + kk * 32) >> 4;
          mma_ss_lo(tbase + 0, kK + off, kQ + off, idSP, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar[B_S]);
      };
      const int ntiles = q_iter().count(a.qpos);
      mbar_wait(&bar[B_KV], 0);
      tc_fence_after();
      if (ntiles > 0) issue_s(0);
      for (int ii = 0; ii < ntiles; ++ii) {
        const int st = ii % QST;
        const uint32_t kQm = desc_lo(smem_u32(smem + Cfg::OFF_Q + st * Cfg::TILE), Cfg::PANEL);
        // dP^T = V dO^T (the dP region must be drained of the previous dQ)
        tl_stamp(a.tl, tlon, 0, ii, 6);
        mbar_wait(&bar[B_DOF], ii & 1);
        tl_stamp(a.tl, tlon, 0, ii, 7);
        if (ii >= 1) mbar_wait(&bar[B_DQE], (ii - 1) & 1);
        tc_fence_after();
        tl_stamp(a.tl, tlon, 0, ii, 0);
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) {
          const int p = k >> 2, kk = k & 3;
          const uint32_t off = (p * Cfg::PANEL + kk * 32) >> 4;
          mma_ss_lo(tbase + 256, kV + off, kDO + off, idSP, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar[B_DP]);
        // dV += P^T dO
        mbar_wait(&bar[B_P], ii & 1);
        tc_fence_after();
        tl_stamp(a.tl, tlon, 0, ii, 1);
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ts_lo(tbase + 128, tbase + 0 + k * 8, kDOm + k * 128, idKV, (ii > 0 || k > 0) ? 1u : 0u);
        mma_commit(&bar[B_DOE]);
        if (ii + 1 < ntiles) issue_s(ii + 1);
        tl_stamp(a.tl, tlon, 0, ii, 2);
        // dQ = dS K (dS as the MN-major A), then dK += dS^T Q (dS as the K-major A)
        mbar_wait(&bar[B_DS], ii & 1);
        tc_fence_after();
        tl_stamp(a.tl, tlon, 0, ii, 3);
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ss_lo(tbase + 256, kDSm + k * 128, kKm + k * 128, idQ, k > 0 ? 1u : 0u);
        mma_commit(&bar[B_DQF]);
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ss_lo(tbase + 384, kDS + (((k >> 2) * Cfg::PANEL + (k & 3) * 32) >> 4), kQm + k * 128, idKV,
                    (ii > 0 || k > 0) ? 1u : 0u);
        mma_commit(&bar[B_QE + st]);
        mma_commit(&bar[B_DSE]);
      }
      mma_commit(&bar[B_DONE]);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ compute: P^T, dS
    // 8 warps: warp w covers TMEM lane quadrant w % 4 (key rows) and query columns
    // [64 h, 64 h + 64), h = (w - 4) / 4.
    const int wq = warp & 3;
    const int hf = (warp - 4) >> 2;
    const int r = wq * 32 + lane;  // key row within the tile
    const uint32_t tl = tbase + (static_cast<uint32_t>(wq * 32) << 16);
    uint8_t* sds = smem + Cfg::OFF_DS + hf * Cfg::PANEL + (r >> 3) * 1024 + (r & 7) * 128;
    int ii = 0;
    int it, qp;
    for (auto iq = q_iter(); iq.next(a.qpos, it, qp);) {
      const int kind = kind_at(qp);
      const int ss = ii & 1;
      const float* slse = stat + ss * 256 + hf * 64;
      const float* sdd = stat + ss * 256 + 128 + hf * 64;
      // stats landed: -lse log2(e) (-inf for query rows with no key at all, so exp2 gives
      // 0 without a branch) and -D / sqrt(d), converted once per call for the packed FMAs
      mbar_wait(&bar[B_SF + ss], (ii >> 1) & 1);
      mbar_wait(&bar[B_S], ii & 1);
      tc_fence_after();
      tl_stamp(a.tl, tlon && threadIdx.x == 128, 1, ii, 0);
      uint32_t pk[32];  // P^T row, this half: 64 bf16
      uint32_t sv[2][32];
      tmem_ld32(tl + hf * 64, sv[0]);
      tmem_ld32(tl + hf * 64 + 32, sv[1]);
      tmem_wait_ld();
      // all of S^T is in registers: P may now overwrite columns [0, 64) (after both warps
      // of this lane quadrant have loaded: the named barrier of the pair), and the dQ drain
      // may park data in [64, 128)
      tc_fence_before();
      mbar_arrive(&bar[B_SL]);
      named_bar_sync(4 + wq, 64);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const uint32_t* rr = sv[c];
        const float2 sc2 = make_float2(a.scale_log2, a.scale_log2);
        if (kind == 2) {  // diagonal tile: key r is visible to query column q iff r <= q
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int q = c * 32 + 2 * i;
            const float2 x = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])), sc2,
                                   *reinterpret_cast<const float2*>(slse + q));
            float e0 = fast_exp2(x.x), e1 = fast_exp2(x.y);
            if (hf * 64 + q < r) e0 = 0.f;
            if (hf * 64 + q + 1 < r) e1 = 0.f;
            pk[c * 16 + i] = pack_bf16x2(e0, e1);
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int q = c * 32 + 2 * i;
            const float2 x = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])), sc2,
                                   *reinterpret_cast<const float2*>(slse + q));
#if WF_BWD_POLY_EVERY > 0
            if ((c * 16 + i) % WF_BWD_POLY_EVERY == WF_BWD_POLY_EVERY - 1) {
              const float2 e = poly_exp2x2(x);
              pk[c * 16 + i] = pack_bf16x2(e.x, e.y);
            } else {
              pk[c * 16 + i] = pack_bf16x2(fast_exp2(x.x), fast_exp2(x.y));
            }
#else
            pk[c * 16 + i] = pack_bf16x2(fast_exp2(x.x), fast_exp2(x.y));
#endif
          }
        }
      }
      tmem_st32(tl + hf * 32, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar[B_P]);
      tl_stamp(a.tl, tlon && threadIdx.x == 128, 1, ii, 1);
      // dS = P o (dP - D), pre-scaled by 1/sqrt(d) for both dK and dQ
      mbar_wait(&bar[B_DP], ii & 1);
      tc_fence_after();
      if (ii >= 1) mbar_wait(&bar[B_DSE], (ii - 1) & 1);  // dQ/dK of tile ii-1 have read dS
      tl_stamp(a.tl, tlon && threadIdx.x == 128, 1, ii, 2);
      uint32_t dk[32];
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t rr[32];
        tmem_ld32(tl + 256 + hf * 64 + c * 32, rr);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 pf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[c * 16 + i]));
          const int q = c * 32 + 2 * i;
          const float2 t = ffma2(make_float2(__uint_as_float(rr[2 * i]), __uint_as_float(rr[2 * i + 1])),
                                 make_float2(a.scale, a.scale), *reinterpret_cast<const float2*>(sdd + q));
          const float2 d = fmul2(pf, t);
          dk[c * 16 + i] = pack_bf16x2(d.x, d.y);
        }
      }
      // dS -> smem (A of both dK and dQ): this half's 64 q = panel hf, row r
#pragma unroll
      for (int j = 0; j < 8; ++j)
        *reinterpret_cast<uint4*>(sds + ((j ^ (r & 7)) << 4)) =
            make_uint4(dk[4 * j], dk[4 * j + 1], dk[4 * j + 2], dk[4 * j + 3]);
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&bar[B_DS]);
      mbar_arrive(&bar[B_SE + ss]);
      tl_stamp(a.tl, tlon && threadIdx.x == 128, 1, ii, 3);
      ++ii;
    }
    // epilogue: dK, dV of this key tile (this warp's half of the 16-column chunks)
    mbar_wait(&bar[B_DONE], 0);
    tc_fence_after();
    const int grow = k0 + r;
    const size_t orow = (static_cast<size_t>(grow) * a.heads + head) * D;
    const bool any = ii > 0;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t col0 = which == 0 ? 384 : 128;
      float* acc = which == 0 ? a.dk_acc : a.dv_acc;
      __nv_bfloat16* outb = which == 0 ? a.dk_out : a.dv_out;
#pragma unroll
      for (int c = hf; c < DP / 16; c += 2) {
        uint32_t rr[16];
        if (any) {
          tmem_ld16(tl + col0 + c * 16, rr);
          tmem_wait_ld();
        }
        float v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) v[i] = any ? __uint_as_float(rr[i]) : 0.f;
        if (c * 16 + 16 <= D) {
          if (outb) {
            uint4* dst = reinterpret_cast<uint4*>(outb + orow + c * 16);
#pragma unroll
            for (int i = 0; i < 2; ++i)
              dst[i] = make_uint4(pack_bf16x2(v[8 * i], v[8 * i + 1]), pack_bf16x2(v[8 * i + 2], v[8 * i + 3]),
                                  pack_bf16x2(v[8 * i + 4], v[8 * i + 5]), pack_bf16x2(v[8 * i + 6], v[8 * i + 7]));
          } else {
            float4* dst = reinterpret_cast<float4*>(acc + orow + c * 16);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              float4 x = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
              if (a.dkv_accumulate) {
                const float4 y = dst[i];
                x.x += y.x;
                x.y += y.y;
                x.z += y.z;
                x.w += y.w;
              }
              dst[i] = x;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const int col = c * 16 + i;
            if (col < D) {
              if (outb)
                outb[orow + col] = __float2bfloat16_rn(v[i]);
              else
                acc[orow + col] = a.dkv_accumulate ? acc[orow + col] + v[i] : v[i];
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ dQ drain (warps 0-3)
    // TMEM -> registers (two 64-column halves; the region is released right after the
    // second half is read) -> this warp's double-buffered staging boxes [32 rows][32 fp32]
    // (128B swizzle, 16-byte chunk j at j ^ (row & 7): conflict-free) -> one TMA tensor
    // reduce-add per box into the fp32 dQ accumulator.
    const uint32_t tl = tbase + (static_cast<uint32_t>(warp * 32) << 16);
    uint8_t* wbox0 = smem + Cfg::OFF_STG + warp * 8192;
    const int ntiles = q_iter().count(a.qpos);
    int ii = 0, chunk = 0;
    int it, qp;
    // read columns [cb, cb + 64) (clipped to DP) of the TMEM address base into ra / rb
    auto ld_half = [&](uint32_t base, int cb, uint32_t(&ra)[32], uint32_t(&rb)[32]) {
      if (cb + 32 <= DP) {
        tmem_ld32(base, ra);
      } else {
        uint32_t r16[16];
        tmem_ld16(base, r16);
#pragma unroll
        for (int i = 0; i < 16; ++i) ra[i] = r16[i];
#pragma unroll
        for (int i = 16; i < 32; ++i) ra[i] = 0u;
      }
      if (cb + 32 < DP) {
        if (cb + 64 <= DP) {
          tmem_ld32(base + 32, rb);
        } else {
          uint32_t r16[16];
          tmem_ld16(base + 32, r16);
#pragma unroll
          for (int i = 0; i < 16; ++i) rb[i] = r16[i];
#pragma unroll
          for (int i = 16; i < 32; ++i) rb[i] = 0u;
        }
      }
    };
    for (auto iq = q_iter(); iq.next(a.qpos, it, qp);) {
      mbar_wait(&bar[B_DQF], ii & 1);
      tc_fence_after();
      tl_stamp(a.tl, tlon && threadIdx.x == 0, 2, ii, 0);
      // Park the second half of dQ in the free columns [64, 128) of the S^T region (the
      // compute warps hold S^T of the next tile in registers by then), so the dP/dQ region
      // is released after two TMEM reads instead of after staging the first half.
      const bool park = kPark && ii + 1 < ntiles;
      if (park) {
        mbar_wait(&bar[B_SL], (ii + 1) & 1);
        tc_fence_after();
        uint32_t ra[32], rb[32];
        ld_half(tl + 256 + 64, 64, ra, rb);
        tmem_wait_ld();
        tmem_st32(tl + 64, ra);
        if (DP > 96) tmem_st32(tl + 96, rb);
      }
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const int cbase = half * 64;
        if (cbase < DP) {
          uint32_t ra[32], rb[32];
          const bool two = cbase + 32 < DP;
          ld_half(half == 1 && park ? tl + 64 : tl + 256 + cbase, cbase, ra, rb);
          tmem_wait_ld();
          if (half == 0 && park) {  // both halves are out of the dP/dQ region
            tmem_wait_st();
            tc_fence_before();
            mbar_arrive(&bar[B_DQE]);
            tl_stamp(a.tl, tlon && threadIdx.x == 0, 2, ii, 1);
          } else if (half == 1 && park) {  // parked half read back: S^T columns free again
            tc_fence_before();
            mbar_arrive(&bar[B_SRF]);
          } else if (cbase + 64 >= DP) {  // last TMEM read of this tile: release the dQ region
            tc_fence_before();
            mbar_arrive(&bar[B_DQE]);
            tl_stamp(a.tl, tlon && threadIdx.x == 0, 2, ii, 1);
          }
#pragma unroll
          for (int sub = 0; sub < 2; ++sub) {
            if (sub == 1 && !two) break;
            const int c0 = cbase + 32 * sub;
            const uint32_t* rr = sub == 0 ? ra : rb;
            uint8_t* wbox = wbox0 + (chunk & 1) * 4096;
            if (lane == 0) bulk_wait_read<1>();  // the reduce of chunk-2 has read this box
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<uint4*>(wbox + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                  make_uint4(rr[4 * j], rr[4 * j + 1], rr[4 * j + 2], rr[4 * j + 3]);
            fence_proxy_async_smem();
            __syncwarp();
            if (lane == 0) {
              tma_reduce_add_3d(&tmDQ, wbox, c0, head, it * WF_TILE + warp * 32);
              bulk_commit();
            }
            ++chunk;
          }
        }
      }
      tl_stamp(a.tl, tlon && threadIdx.x == 0, 2, ii, 2);
      ++ii;
    }
    if (lane == 0) bulk_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 13) tmem_dealloc(tbase, 512);
}

template <int D>
cudaError_t launch_bwd_d(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const CUtensorMap& tdo, const CUtensorMap& tdq, const BwdArgs& a, cudaStream_t s) {
  using Cfg = BwdCfg<D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(wf_block_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(a.nk / WF_TILE, a.heads);
  BwdArgs b = a;
  b.tl = timeline_buffer();
  b.tl_cta = timeline_cta();
  wf_block_bwd_kernel<D><<<grid, kThreads, Cfg::SMEM, s>>>(tq, tk, tv, tdo, tdq, b);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_block_bwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                             const CUtensorMap& tdo, const BwdArgs& a, int D, cudaStream_t s) {
  if (a.nq % WF_TILE || a.nk <= 0 || a.nk % WF_TILE) return cudaErrorInvalidValue;
  CUtensorMap tdq;
  if (!make_tmap_f32_rows(&tdq, a.dq_acc, a.nq > 0 ? a.nq : WF_TILE, a.heads, D)) return cudaErrorInvalidValue;
  switch (D) {
    case 128: return launch_bwd_d<128>(tq, tk, tv, tdo, tdq, a, s);
    case 64: return launch_bwd_d<64>(tq, tk, tv, tdo, tdq, a, s);
    case 72: return launch_bwd_d<72>(tq, tk, tv, tdo, tdq, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace wf
