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
// 10 warps: 0-3 dQ drain (TMEM -> fp32 atomics, lane = query row), 4-7 compute
// (lane = key row), 8 TMA producer, 9 TMEM allocator + MMA issuer.
// TMEM: S^T [0,128) (P^T bf16 over [0,64)), dV [128,128+DP), dP^T [256,384)
// (dS^T bf16 over [256,320), then dQ over [256,256+DP)), dK [384,384+DP).
#include "common.h"
#include "sm100.cuh"

namespace wf {
using namespace sm100;

namespace {

constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ int tile_gpos(const PosTable& t, int row0) {
  return t.start[row0 / t.chunk] + row0 % t.chunk;
}

// for K tile at kpos0: 0 = q tile fully masked, 1 = full, 2 = diagonal
__device__ __forceinline__ int qtile_kind(const BwdArgs& a, int kpos0, int it) {
  if (!a.causal) return 1;
  const int qp0 = tile_gpos(a.qpos, it * WF_TILE);
  return qp0 < kpos0 ? 0 : (qp0 == kpos0 ? 2 : 1);
}

template <int D>
struct BwdCfg {
  static constexpr int DP = (D + 15) / 16 * 16;
  static constexpr int NP = (D + 63) / 64;
  static constexpr int PANEL = 128 * 128;
  static constexpr int TILE = NP * PANEL;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = TILE;
  static constexpr int OFF_Q = 2 * TILE;        // 2 stages
  static constexpr int OFF_DO = 4 * TILE;       // 1 stage
  static constexpr int OFF_DS = 5 * TILE;       // [128 q] x [128 kv] bf16, MN-major SW128 (2 panels)
  static constexpr int OFF_STAT = OFF_DS + 2 * PANEL;  // 2 stages x (lse[128], dsum[128]) fp32
  static constexpr int OFF_BAR = OFF_STAT + 2 * 1024;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;
};

enum {
  B_KV = 0, B_QF = 1, B_QE = 3, B_DOF = 5, B_DOE = 6, B_S = 7, B_DP = 8, B_P = 9, B_DS = 10, B_DQF = 11,
  B_DQE = 12, B_DSE = 13, B_DONE = 14, B_NUM = 15
};

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

template <int D>
__global__ void __maxnreg__(200)
    wf_block_bwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmDO,
                        const __grid_constant__ BwdArgs a) {
  using Cfg = BwdCfg<D>;
  constexpr int DP = Cfg::DP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + B_NUM * 8);
  float* stat = reinterpret_cast<float*>(smem + Cfg::OFF_STAT);  // [stage][2][128]

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int kt = blockIdx.x;
  const int head = blockIdx.y;
  const int k0 = kt * WF_TILE;
  const int kpos0 = a.causal ? tile_gpos(a.kpos, k0) : k0;
  const int nqt = a.nq / WF_TILE;

  if (threadIdx.x == 0) {
    mbar_init(&bar[B_KV], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[B_QF + i], 1);
      mbar_init(&bar[B_QE + i], 1);
    }
    mbar_init(&bar[B_DOF], 1);
    mbar_init(&bar[B_DOE], 1);
    mbar_init(&bar[B_S], 1);
    mbar_init(&bar[B_DP], 1);
    mbar_init(&bar[B_P], 128);
    mbar_init(&bar[B_DS], 128);
    mbar_init(&bar[B_DQF], 1);
    mbar_init(&bar[B_DQE], 128);
    mbar_init(&bar[B_DSE], 1);
    mbar_init(&bar[B_DONE], 1);
    fence_barrier_init();
  }
  if (warp == 9) {
    tmem_alloc(tmem_slot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tmem_slot;

  if (warp == 8) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      tma_prefetch_desc(&tmDO);
      mbar_arrive_expect_tx(&bar[B_KV], 2 * Cfg::TILE);
      for (int p = 0; p < Cfg::NP; ++p) {
        tma_load_3d(smem + Cfg::OFF_K + p * Cfg::PANEL, &tmK, &bar[B_KV], p * 64, head, k0);
        tma_load_3d(smem + Cfg::OFF_V + p * Cfg::PANEL, &tmV, &bar[B_KV], p * 64, head, k0);
      }
      int ii = 0;
      for (int it = 0; it < nqt; ++it) {
        if (qtile_kind(a, kpos0, it) == 0) continue;
        const int st = ii & 1;
        if (ii >= 2) mbar_wait(&bar[B_QE + st], ((ii - 2) >> 1) & 1);
        mbar_arrive_expect_tx(&bar[B_QF + st], Cfg::TILE + 1024);
        for (int p = 0; p < Cfg::NP; ++p)
          tma_load_3d(smem + Cfg::OFF_Q + st * Cfg::TILE + p * Cfg::PANEL, &tmQ, &bar[B_QF + st], p * 64, head,
                      it * WF_TILE);
        const int64_t soff = stat_index(head, it * WF_TILE, a.heads, a.stat_blk);
        bulk_load(stat + st * 256, a.lse + soff, 512, &bar[B_QF + st]);
        bulk_load(stat + st * 256 + 128, a.dsum + soff, 512, &bar[B_QF + st]);
        if (ii >= 1) mbar_wait(&bar[B_DOE], (ii - 1) & 1);
        mbar_arrive_expect_tx(&bar[B_DOF], Cfg::TILE);
        for (int p = 0; p < Cfg::NP; ++p)
          tma_load_3d(smem + Cfg::OFF_DO + p * Cfg::PANEL, &tmDO, &bar[B_DOF], p * 64, head, it * WF_TILE);
        ++ii;
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idSP = idesc_bf16_f32(128, 128, 0, 0);   // K x Q^T, V x dO^T (both K-major)
      constexpr uint32_t idKV = idesc_bf16_f32(128, DP, 0, 1);    // P^T/dS^T (TMEM) x dO/Q (MN-major)
      constexpr uint32_t idQ = idesc_bf16_f32(128, DP, 1, 1);     // dS (smem, MN-major) x K (MN-major)
      const uint32_t sK = smem_u32(smem + Cfg::OFF_K);
      const uint32_t sV = smem_u32(smem + Cfg::OFF_V);
      const uint32_t sDO = smem_u32(smem + Cfg::OFF_DO);
      const uint32_t sDS = smem_u32(smem + Cfg::OFF_DS);
      mbar_wait(&bar[B_KV], 0);
      tc_fence_after();
      int ii = 0;
      for (int it = 0; it < nqt; ++it) {
        if (qtile_kind(a, kpos0, it) == 0) continue;
        const int st = ii & 1;
        const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q + st * Cfg::TILE);
        // S^T = K Q^T
        mbar_wait(&bar[B_QF + st], (ii >> 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) {
          const int p = k >> 2, kk = k & 3;
          mma_ss(tbase + 0, smem_desc_sw128(sK + p * Cfg::PANEL + kk * 32, 16, 1024),
                 smem_desc_sw128(sQ + p * Cfg::PANEL + kk * 32, 16, 1024), idSP, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar[B_S]);
        // dP^T = V dO^T  (dP region must be drained of the previous dQ)
        mbar_wait(&bar[B_DOF], ii & 1);
        if (ii >= 1) mbar_wait(&bar[B_DQE], (ii - 1) & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) {
          const int p = k >> 2, kk = k & 3;
          mma_ss(tbase + 256, smem_desc_sw128(sV + p * Cfg::PANEL + kk * 32, 16, 1024),
                 smem_desc_sw128(sDO + p * Cfg::PANEL + kk * 32, 16, 1024), idSP, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar[B_DP]);
        // dV += P^T dO
        mbar_wait(&bar[B_P], ii & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ts(tbase + 128, tbase + 0 + k * 8, smem_desc_sw128(sDO + k * 2048, Cfg::PANEL, 1024), idKV,
                 (ii > 0 || k > 0) ? 1u : 0u);
        mma_commit(&bar[B_DOE]);
        // dK += dS^T Q ; dQ = dS K
        mbar_wait(&bar[B_DS], ii & 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ts(tbase + 384, tbase + 256 + k * 8, smem_desc_sw128(sQ + k * 2048, Cfg::PANEL, 1024), idKV,
                 (ii > 0 || k > 0) ? 1u : 0u);
        mma_commit(&bar[B_QE + st]);
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k)
          mma_ss(tbase + 256, smem_desc_sw128(sDS + k * 2048, Cfg::PANEL, 1024),
                 smem_desc_sw128(sK + k * 2048, Cfg::PANEL, 1024), idQ, k > 0 ? 1u : 0u);
        mma_commit(&bar[B_DQF]);
        mma_commit(&bar[B_DSE]);
        ++ii;
      }
      mma_commit(&bar[B_DONE]);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ compute: P^T, dS^T
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // key row within the tile
    const uint32_t tl = tbase + (static_cast<uint32_t>(wq * 32) << 16);
    uint8_t* sds = smem + Cfg::OFF_DS;
    int ii = 0;
    for (int it = 0; it < nqt; ++it) {
      const int kind = qtile_kind(a, kpos0, it);
      if (kind == 0) continue;
      const int st = ii & 1;
      const float* slse = stat + st * 256;
      const float* sdd = slse + 128;
      mbar_wait(&bar[B_QF + st], (ii >> 1) & 1);  // stats landed
      mbar_wait(&bar[B_S], ii & 1);
      tc_fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32];
        tmem_ld32(tl + c * 32, rr);
        tmem_wait_ld();
        float p[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const int q = c * 32 + i;
          const float lq = slse[q];
          float e = fast_exp2(fmaf(__uint_as_float(rr[i]), a.scale_log2, -lq * kLog2e));
          if (lq == -INFINITY || (kind == 2 && q < r)) e = 0.f;
          p[i] = e;
        }
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) pk[i] = pack_bf16x2(p[2 * i], p[2 * i + 1]);
        tmem_st16(tl + c * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar[B_P]);
      // dS^T = P^T o (dP^T - D)
      mbar_wait(&bar[B_DP], ii & 1);
      tc_fence_after();
      // dS^T -> TMEM (A of dK += dS^T Q), dS -> smem (A of dQ = dS K, MN-major).
      // P^T is re-read as the bf16 copy already in TMEM (keeps 128 fp32 registers free).
      if (ii >= 1) mbar_wait(&bar[B_DSE], (ii - 1) & 1);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t rr[32], pb[16];
        tmem_ld32(tl + 256 + c * 32, rr);
        tmem_ld16(tl + c * 16, pb);
        tmem_wait_ld();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float2 pf = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pb[i]));
          const float d0 = pf.x * (__uint_as_float(rr[2 * i]) - sdd[c * 32 + 2 * i]);
          const float d1 = pf.y * (__uint_as_float(rr[2 * i + 1]) - sdd[c * 32 + 2 * i + 1]);
          pk[i] = pack_bf16x2(d0, d1);
        }
        tmem_st16(tl + 256 + c * 16, pk);
        // 32 q values = 4 chunks of 16 B in panel (c >> 1), chunks (c & 1) * 4 + j
        uint8_t* rowp = sds + (c >> 1) * Cfg::PANEL + (r >> 3) * 1024 + (r & 7) * 128;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const int chunk = (c & 1) * 4 + j;
          *reinterpret_cast<uint4*>(rowp + ((chunk ^ (r & 7)) << 4)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
      }
      fence_proxy_async_smem();
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar[B_DS]);
      ++ii;
    }
    // epilogue: dK (scaled), dV of this key tile
    mbar_wait(&bar[B_DONE], 0);
    tc_fence_after();
    const int grow = k0 + r;
    const size_t orow = (static_cast<size_t>(grow) * a.heads + head) * D;
    const bool any = ii > 0;
#pragma unroll
    for (int which = 0; which < 2; ++which) {
      const uint32_t col0 = which == 0 ? 384 : 128;
      const float sc = which == 0 ? a.scale : 1.f;
      float* acc = which == 0 ? a.dk_acc : a.dv_acc;
      __nv_bfloat16* outb = which == 0 ? a.dk_out : a.dv_out;
#pragma unroll
      for (int c = 0; c < DP / 16; ++c) {
        uint32_t rr[16];
        if (any) {
          tmem_ld16(tl + col0 + c * 16, rr);
          tmem_wait_ld();
        }
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int col = c * 16 + i;
          if (col < D) {
            const float v = any ? __uint_as_float(rr[i]) * sc : 0.f;
            if (outb) {
              outb[orow + col] = __float2bfloat16_rn(v);
            } else if (acc) {
              acc[orow + col] = a.dkv_accumulate ? acc[orow + col] + v : v;
            }
          }
        }
      }
    }
  } else {
    // ------------------------------------------------------------ dQ drain (warps 0-3)
    const int r = warp * 32 + lane;  // query row within the tile
    const uint32_t tl = tbase + (static_cast<uint32_t>(warp * 32) << 16);
    int ii = 0;
    for (int it = 0; it < nqt; ++it) {
      if (qtile_kind(a, kpos0, it) == 0) continue;
      mbar_wait(&bar[B_DQF], ii & 1);
      tc_fence_after();
      float* dst = a.dq_acc + (static_cast<size_t>(it * WF_TILE + r) * a.heads + head) * D;
#pragma unroll
      for (int c = 0; c < DP / 16; ++c) {
        uint32_t rr[16];
        tmem_ld16(tl + 256 + c * 16, rr);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (c * 16 + 4 * j < D)
            atomicAdd(reinterpret_cast<float4*>(dst + c * 16) + j,
                      make_float4(__uint_as_float(rr[4 * j]) * a.scale, __uint_as_float(rr[4 * j + 1]) * a.scale,
                                  __uint_as_float(rr[4 * j + 2]) * a.scale, __uint_as_float(rr[4 * j + 3]) * a.scale));
      }
      tc_fence_before();
      mbar_arrive(&bar[B_DQE]);
      ++ii;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc(tbase, 512);
}

template <int D>
cudaError_t launch_bwd_d(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                         const CUtensorMap& tdo, const BwdArgs& a, cudaStream_t s) {
  using Cfg = BwdCfg<D>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(wf_block_bwd_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid(a.nk / WF_TILE, a.heads);
  wf_block_bwd_kernel<D><<<grid, 320, Cfg::SMEM, s>>>(tq, tk, tv, tdo, a);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_block_bwd(const CUtensorMap& tq, const CUtensorMap& tk, const CUtensorMap& tv,
                             const CUtensorMap& tdo, const BwdArgs& a, int D, cudaStream_t s) {
  if (a.nq % WF_TILE || a.nk <= 0 || a.nk % WF_TILE) return cudaErrorInvalidValue;
  switch (D) {
    case 128: return launch_bwd_d<128>(tq, tk, tv, tdo, a, s);
    case 64: return launch_bwd_d<64>(tq, tk, tv, tdo, a, s);
    case 72: return launch_bwd_d<72>(tq, tk, tv, tdo, a, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace wf
