// gemm.cu -- Y = A B^T in bf16 on tcgen05 for the QKV projection (Alg. 1 l.1,
// "AllGather_QKVmatmul"), with a multi-destination epilogue: each output tile is written
// to the caller's Q/K/V and, when fused, straight into the team members' gathered buffers
// over NVLink peer memory, so the team all-gather rides on the GEMM's
// epilogue instead of a separate copy phase.
//
// Persistent CTAs (one per SM) walk a static tile schedule (bands of 16 M-tiles across all
// N-tiles, so the tiles in flight share their A and B panels in L2).  6 warps: warp 0 TMA
// producer (4-stage ring of [128 x 64] A and [BN x 64] B SW128 boxes), warp 1 TMEM
// allocator + single-thread MMA issuer (M = 128, N = BN, fp32 accumulators double-buffered
// in TMEM so the epilogue of tile i overlaps the main loop of tile i+1), warps 2-5 the
// epilogue (TMEM lane quadrant = 32 output rows; 32-column chunks -> bf16 -> a swizzled
// shared staging box -> coalesced 16-byte stores to every destination).
#include <cstdlib>

#include "common.h"
#include "sm100.cuh"

namespace wf {
using namespace sm100;

namespace {

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128, BK = 64, ST = 4;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int OFF_STG = ST * STAGE;           // 4 warps x 2 x [32 rows x 64 B]
  static constexpr int OFF_BAR = OFF_STG + 4 * 4096;
  static constexpr int SMEM = OFF_BAR + 256;
  static constexpr int TCOLS = 2 * BN;
  static_assert(SMEM <= 232448, "shared memory budget");
};
enum { G_FULL = 0, G_EMPTY = 4, G_TFULL = 8, G_TEMPTY = 10, G_NUM = 12 };

// tile -> (m, n): bands of 16 M-tiles sweep all N-tiles
__device__ __forceinline__ void tile_coords(int tile, int nm, int nn, int& m, int& n) {
  constexpr int kBand = 16;
  const int per_band = kBand * nn;
  const int b = tile / per_band, r = tile - b * per_band;
  const int rows = min(kBand, nm - b * kBand);
  m = b * kBand + r % rows;
  n = r / rows;
}

// A_MN / B_MN: operand stored MN-major ([K, M] / [K, N] row-major: the transposed operands
// of the backward GEMMs dX = dY W and dW = dY^T X) instead of K-major ([M, K] / [N, K]).
// MN-major tiles arrive as 64-column panels of [64 K rows x 128 B] (8 KB), LBO = 8 KB.
template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(192, 1)
    wf_gemm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                   const __grid_constant__ GemmArgs g) {
  using Cfg = GemmCfg<BN>;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + G_NUM * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nm = g.M / 128, nn = g.N / BN, ntiles = nm * nn, nk = g.K / 64;

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    for (int i = 0; i < Cfg::ST; ++i) {
      mbar_init(&bar[G_FULL + i], 1);
      mbar_init(&bar[G_EMPTY + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[G_TFULL + i], 1);
      mbar_init(&bar[G_TEMPTY + i], 4);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc(tslot, Cfg::TCOLS);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(&tB);
      int it = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        int m, n;
        tile_coords(tile, nm, nn, m, n);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % Cfg::ST;
          if (it >= Cfg::ST) mbar_wait(&bar[G_EMPTY + s], ((it / Cfg::ST) - 1) & 1);
          uint8_t* sa = smem + s * Cfg::STAGE;
          mbar_arrive_expect_tx(&bar[G_FULL + s], Cfg::STAGE);
          if (A_MN) {
            for (int p = 0; p < 2; ++p) tma_load_2d(sa + p * 8192, &tA, &bar[G_FULL + s], m * 128 + p * 64, kb * 64);
          } else {
            tma_load_2d(sa, &tA, &bar[G_FULL + s], kb * 64, m * 128);
          }
          if (B_MN) {
            for (int p = 0; p < BN / 64; ++p)
              tma_load_2d(sa + Cfg::A_BYTES + p * 8192, &tB, &bar[G_FULL + s], n * BN + p * 64, kb * 64);
          } else {
            tma_load_2d(sa + Cfg::A_BYTES, &tB, &bar[G_FULL + s], kb * 64, n * BN);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(128, BN, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int it = 0, lt = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
        const int b = lt & 1;
        if (lt >= 2) mbar_wait(&bar[G_TEMPTY + b], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tbase + b * BN;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % Cfg::ST;
          mbar_wait(&bar[G_FULL + s], (it / Cfg::ST) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * Cfg::STAGE), sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = A_MN ? smem_desc_sw128(sa + kk * 2048, 8192, 1024) : smem_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? smem_desc_sw128(sb + kk * 2048, 8192, 1024) : smem_desc_sw128(sb + kk * 32, 16, 1024);
            mma_ss(acc, da, db, idesc, (kb | kk) ? 1u : 0u);
          }
          mma_commit(&bar[G_EMPTY + s]);
        }
        mma_commit(&bar[G_TFULL + b]);
      }
    }
  } else {
    // epilogue: warps 2..5 own TMEM lane quadrants 2, 3, 0, 1
    const int q = warp & 3;
    const uint32_t tl = tbase + (static_cast<uint32_t>(q * 32) << 16);
    uint8_t* stg = smem + Cfg::OFF_STG + (warp - 2) * 4096;
    int lt = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++lt) {
      int m, n;
      tile_coords(tile, nm, nn, m, n);
      const int b = lt & 1;
      const int c0 = n * BN;
      const int part = c0 / g.split;
      const int pc0 = c0 - part * g.split;
      __nv_bfloat16* dp[WF_GEMM_MAX_DST];
#pragma unroll
      for (int d = 0; d < WF_GEMM_MAX_DST; ++d)
        dp[d] = part == 0 ? g.out[0][d] : (part == 1 ? g.out[1][d] : g.out[2][d]);
      const int nd = part == 0 ? g.ndst[0] : (part == 1 ? g.ndst[1] : g.ndst[2]);
      mbar_wait(&bar[G_TFULL + b], (lt >> 1) & 1);
      tc_fence_after();
      const int64_t rowbase = static_cast<int64_t>(m) * 128 + q * 32;
#pragma unroll 1
      for (int ch = 0; ch < BN / 32; ++ch) {
        uint32_t r[32];
        tmem_ld32(tl + b * BN + ch * 32, r);
        tmem_wait_ld();
        uint8_t* sb = stg + (ch & 1) * 2048;
        // row = lane: 64 B as four 16-B granules, XOR-swizzled by (row >> 1) & 3 (no bank conflicts)
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) {
          const uint4 v = make_uint4(pack_bf16x2(__uint_as_float(r[8 * gq + 0]), __uint_as_float(r[8 * gq + 1])),
                                     pack_bf16x2(__uint_as_float(r[8 * gq + 2]), __uint_as_float(r[8 * gq + 3])),
                                     pack_bf16x2(__uint_as_float(r[8 * gq + 4]), __uint_as_float(r[8 * gq + 5])),
                                     pack_bf16x2(__uint_as_float(r[8 * gq + 6]), __uint_as_float(r[8 * gq + 7])));
          *reinterpret_cast<uint4*>(sb + lane * 64 + ((gq ^ ((lane >> 1) & 3)) << 4)) = v;
        }
        __syncwarp();
        // coalesced copy-out: each instruction stores 8 rows x 64 B
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i * 8 + (lane >> 2), gq = lane & 3;
          const uint4 v = *reinterpret_cast<const uint4*>(sb + row * 64 + ((gq ^ ((row >> 1) & 3)) << 4));
          const int64_t off = (rowbase + row) * g.ld + pc0 + ch * 32 + gq * 8;
#pragma unroll
          for (int d = 0; d < WF_GEMM_MAX_DST; ++d)
            if (d < nd) *reinterpret_cast<uint4*>(dp[d] + off) = v;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bar[G_TEMPTY + b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tbase, Cfg::TCOLS);
}

// ---------------------------------------------------------------- CTA-pair variant
// Same contract for every operand layout (K- or MN-major A and B), pair tile 256 x 256: the even CTA of a cluster of two
// issues M = 256 `tcgen05.mma.cta_group::2` MMAs whose A rows [0, 128) come from its own
// shared memory and [128, 256) from its peer's, with the 256 N rows of B split 128 / 128;
// each CTA loads half of both operand tiles and receives its 128 output rows x 256 columns
// in its own TMEM.  Per SM that is 3/4 of the operand traffic of the 128 x 256 tile.  TMA
// completion of both CTAs is counted on the even CTA's full barrier; its MMA commits are
// multicast to both CTAs' empty / accumulator barriers; both epilogues release the
// accumulator on the even CTA's barrier.
struct Gemm2Cfg {
  static constexpr int ST = 6;
  static constexpr int A_BYTES = 128 * 64 * 2;
  static constexpr int B_BYTES = 128 * 64 * 2;
  static constexpr int STAGE = A_BYTES + B_BYTES;
  static constexpr int OFF_STG = ST * STAGE;
  static constexpr int OFF_BAR = OFF_STG + 4 * 4096;
  static constexpr int SMEM = OFF_BAR + 256;
  static_assert(SMEM <= 232448, "shared memory budget");
};
enum { P_FULL = 0, P_EMPTY = 6, P_TFULL = 12, P_TEMPTY = 14, P_NUM = 16 };

template <bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
    wf_gemm2_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB,
                    const __grid_constant__ GemmArgs g) {
  using Cfg = Gemm2Cfg;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + P_NUM * 8);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  const int nm = g.M / 256, nn = g.N / 256, ntiles = nm * nn, nk = g.K / 64;

  if (threadIdx.x == 0) {
    if (smem_u32(smem) & 1023) __trap();
    for (int i = 0; i < Cfg::ST; ++i) {
      mbar_init(&bar[P_FULL + i], 1);
      mbar_init(&bar[P_EMPTY + i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[P_TFULL + i], 1);
      mbar_init(&bar[P_TEMPTY + i], 8);  // 4 epilogue warps x 2 CTAs
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    tmem_alloc2(tslot, 512);
    tmem_relinquish2();
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tbase = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      tma_prefetch_desc(&tA);
      tma_prefetch_desc(&tB);
      int it = 0;
      for (int tile = cid; tile < ntiles; tile += ncl) {
        int m, n;
        tile_coords(tile, nm, nn, m, n);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % Cfg::ST;
          if (it >= Cfg::ST) mbar_wait(&bar[P_EMPTY + s], ((it / Cfg::ST) - 1) & 1);
          uint8_t* sa = smem + s * Cfg::STAGE;
          if (cr == 0) mbar_arrive_expect_tx(&bar[P_FULL + s], 2 * Cfg::STAGE);
          // this CTA's 128 rows of A (M) and of B (N); MN-major operands as two 64-column panels
          if (A_MN) {
            for (int p = 0; p < 2; ++p)
              tma_load_2d_pair(sa + p * 8192, &tA, &bar[P_FULL + s], m * 256 + cr * 128 + p * 64, kb * 64);
          } else {
            tma_load_2d_pair(sa, &tA, &bar[P_FULL + s], kb * 64, m * 256 + cr * 128);
          }
          if (B_MN) {
            for (int p = 0; p < 2; ++p)
              tma_load_2d_pair(sa + Cfg::A_BYTES + p * 8192, &tB, &bar[P_FULL + s], n * 256 + cr * 128 + p * 64,
                               kb * 64);
          } else {
            tma_load_2d_pair(sa + Cfg::A_BYTES, &tB, &bar[P_FULL + s], kb * 64, n * 256 + cr * 128);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (cr == 0 && lane == 0) {
      constexpr uint32_t idesc = idesc_bf16_f32(256, 256, A_MN ? 1 : 0, B_MN ? 1 : 0);
      int it = 0, lt = 0;
      for (int tile = cid; tile < ntiles; tile += ncl, ++lt) {
        const int b = lt & 1;
        if (lt >= 2) mbar_wait(&bar[P_TEMPTY + b], ((lt >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t acc = tbase + b * 256;
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % Cfg::ST;
          mbar_wait(&bar[P_FULL + s], (it / Cfg::ST) & 1);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + s * Cfg::STAGE), sb = sa + Cfg::A_BYTES;
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            const uint64_t da = A_MN ? smem_desc_sw128(sa + kk * 2048, 8192, 1024) : smem_desc_sw128(sa + kk * 32, 16, 1024);
            const uint64_t db = B_MN ? smem_desc_sw128(sb + kk * 2048, 8192, 1024) : smem_desc_sw128(sb + kk * 32, 16, 1024);
            mma2_ss(acc, da, db, idesc, (kb | kk) ? 1u : 0u);
          }
          mma2_commit_mc(&bar[P_EMPTY + s], 0x3);
        }
        mma2_commit_mc(&bar[P_TFULL + b], 0x3);
      }
    }
  } else {
    const int q = warp & 3;
    const uint32_t tl = tbase + (static_cast<uint32_t>(q * 32) << 16);
    uint8_t* stg = smem + Cfg::OFF_STG + (warp - 2) * 4096;
    int lt = 0;
    for (int tile = cid; tile < ntiles; tile += ncl, ++lt) {
      int m, n;
      tile_coords(tile, nm, nn, m, n);
      const int b = lt & 1;
      const int c0 = n * 256;
      const int part = c0 / g.split;
      const int pc0 = c0 - part * g.split;
      __nv_bfloat16* dp[WF_GEMM_MAX_DST];
#pragma unroll
      for (int d = 0; d < WF_GEMM_MAX_DST; ++d)
        dp[d] = part == 0 ? g.out[0][d] : (part == 1 ? g.out[1][d] : g.out[2][d]);
      const int nd = part == 0 ? g.ndst[0] : (part == 1 ? g.ndst[1] : g.ndst[2]);
      mbar_wait(&bar[P_TFULL + b], (lt >> 1) & 1);
      tc_fence_after();
      const int64_t rowbase = static_cast<int64_t>(m) * 256 + cr * 128 + q * 32;
#pragma unroll 1
      for (int ch = 0; ch < 8; ++ch) {
        uint32_t r[32];
        tmem_ld32(tl + b * 256 + ch * 32, r);
        tmem_wait_ld();
        uint8_t* sb = stg + (ch & 1) * 2048;
#pragma unroll
        for (int gq = 0; gq < 4; ++gq) {
          const uint4 v = make_uint4(pack_bf16x2(__uint_as_float(r[8 * gq + 0]), __uint_as_float(r[8 * gq + 1])),
                                     pack_bf16x2(__uint_as_float(r[8 * gq + 2]), __uint_as_float(r[8 * gq + 3])),
                                     pack_bf16x2(__uint_as_float(r[8 * gq + 4]), __uint_as_float(r[8 * gq + 5])),
                                     pack_bf16x2(__uint_as_float(r[8 * gq + 6]), __uint_as_float(r[8 * gq + 7])));
          *reinterpret_cast<uint4*>(sb + lane * 64 + ((gq ^ ((lane >> 1) & 3)) << 4)) = v;
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int row = i * 8 + (lane >> 2), gq = lane & 3;
          const uint4 v = *reinterpret_cast<const uint4*>(sb + row * 64 + ((gq ^ ((row >> 1) & 3)) << 4));
          const int64_t off = (rowbase + row) * g.ld + pc0 + ch * 32 + gq * 8;
#pragma unroll
          for (int d = 0; d < WF_GEMM_MAX_DST; ++d)
            if (d < nd) *reinterpret_cast<uint4*>(dp[d] + off) = v;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(&bar[P_TEMPTY + b], 0);
    }
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 1) tmem_dealloc2(tbase, 512);
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, bool A_MN, bool B_MN>
cudaError_t launch_bn(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, cudaStream_t s) {
  using Cfg = GemmCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(wf_gemm_kernel<BN, A_MN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int ntiles = (g.M / 128) * (g.N / BN);
  const int grid = ntiles < sm_count() ? ntiles : sm_count();
  wf_gemm_kernel<BN, A_MN, B_MN><<<grid, 192, Cfg::SMEM, s>>>(ta, tb, g);
  return cudaGetLastError();
}

template <int BN>
cudaError_t launch_layout(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int a_mn, int b_mn,
                          cudaStream_t s) {
  if (!a_mn && !b_mn) return launch_bn<BN, false, false>(ta, tb, g, s);
  if (!a_mn && b_mn) return launch_bn<BN, false, true>(ta, tb, g, s);
  if (a_mn && b_mn) return launch_bn<BN, true, true>(ta, tb, g, s);
  return launch_bn<BN, true, false>(ta, tb, g, s);
}

}  // namespace

cudaError_t launch_gemm(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int bn, cudaStream_t s) {
  return launch_gemm_t(ta, tb, g, bn, 0, 0, s);
}

bool gemm_pair_ok(const GemmArgs& g, int /*a_mn*/, int /*b_mn*/) {
  return g.M % 256 == 0 && g.N % 256 == 0 && g.split % 256 == 0;
}

namespace {
template <bool A_MN, bool B_MN>
cudaError_t launch_pair_layout(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, cudaStream_t s) {
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(wf_gemm2_kernel<A_MN, B_MN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Gemm2Cfg::SMEM);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int ntiles = (g.M / 256) * (g.N / 256);
  const int pairs = ntiles < sm_count() / 2 ? ntiles : sm_count() / 2;
  wf_gemm2_kernel<A_MN, B_MN><<<2 * pairs, 192, Gemm2Cfg::SMEM, s>>>(ta, tb, g);
  return cudaGetLastError();
}
}  // namespace

cudaError_t launch_gemm_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int a_mn, int b_mn,
                             cudaStream_t s) {
  if (!a_mn && !b_mn) return launch_pair_layout<false, false>(ta, tb, g, s);
  if (!a_mn && b_mn) return launch_pair_layout<false, true>(ta, tb, g, s);
  if (a_mn && b_mn) return launch_pair_layout<true, true>(ta, tb, g, s);
  return launch_pair_layout<true, false>(ta, tb, g, s);
}

cudaError_t launch_gemm_t(const CUtensorMap& ta, const CUtensorMap& tb, const GemmArgs& g, int bn, int a_mn, int b_mn,
                          cudaStream_t s) {
  if (g.M <= 0 || g.M % 128 || g.K <= 0 || g.K % 64 || g.N <= 0 || g.N % bn || g.split % bn)
    return cudaErrorInvalidValue;
  for (int p = 0; p < 3; ++p)
    if (g.ndst[p] < 0 || g.ndst[p] > WF_GEMM_MAX_DST) return cudaErrorInvalidValue;
  switch (bn) {
    case 256: return launch_layout<256>(ta, tb, g, a_mn, b_mn, s);
    case 128: return launch_layout<128>(ta, tb, g, a_mn, b_mn, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace wf
