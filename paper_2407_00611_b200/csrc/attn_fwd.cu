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
// CTA = 6 warps: warp 0 TMA producer, warp 1 TMEM allocator + single-thread MMA
// issuer, warps 2..5 softmax/epilogue (thread <-> TMEM lane <-> query row).
// TMEM: S double buffer at cols [0,128) and [128,256); O at [256, 256+DP).
#include "common.h"
#include "sm100.cuh"

namespace wf {
using namespace sm100;

namespace {

constexpr float kLog2e = 1.4426950408889634f;
constexpr float kLn2 = 0.6931471805599453f;

__device__ __forceinline__ int tile_gpos(const PosTable& t, int row0) {
  return t.start[row0 / t.chunk] + row0 % t.chunk;
}

// 0 = fully masked (skip), 1 = fully visible, 2 = diagonal
__device__ __forceinline__ int tile_kind(const FwdArgs& a, int qpos0, int jt) {
  if (!a.causal) return 1;
  int kp0 = tile_gpos(a.kpos, jt * WF_TILE);
  return kp0 > qpos0 ? 0 : (kp0 == qpos0 ? 2 : 1);
}

template <int D>
struct FwdCfg {
  static constexpr int DP = (D + 15) / 16 * 16;   // MMA-padded head dim
  static constexpr int NP = (D + 63) / 64;        // 64-column smem panels per tile
  static constexpr int PANEL = 128 * 128;         // bytes of one [128 rows x 64 bf16] panel
  static constexpr int TILE = NP * PANEL;
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = TILE;
  static constexpr int OFF_V = 3 * TILE;
  static constexpr int OFF_BAR = 5 * TILE;
  static constexpr int SMEM = OFF_BAR + 256 + 1024;  // + alignment slack
};

enum { B_Q = 0, B_K = 1, B_V = 3, B_KVE = 5, B_S = 7, B_P = 9, B_O = 11, B_NUM = 12 };

template <int D>
__global__ void __launch_bounds__(192, 1)
    wf_block_fwd_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                        const __grid_constant__ CUtensorMap tmV, const __grid_constant__ FwdArgs a) {
  using Cfg = FwdCfg<D>;
  constexpr int DP = Cfg::DP;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Cfg::OFF_BAR);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + Cfg::OFF_BAR + B_NUM * 8);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nqt = a.nq / WF_TILE;
  // heavy tiles first: with zigzag units the later half of each unit sees more keys
  const int qt = a.causal ? (nqt - 1 - blockIdx.x) : blockIdx.x;
  const int head = blockIdx.y;
  const int q0 = qt * WF_TILE;
  const int qpos0 = a.causal ? tile_gpos(a.qpos, q0) : q0;
  const int nkt = a.nk / WF_TILE;
  const bool has_state = a.o_in != nullptr;

  if (threadIdx.x == 0) {
    mbar_init(&bar[B_Q], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar[B_K + i], 1);
      mbar_init(&bar[B_V + i], 1);
      mbar_init(&bar[B_KVE + i], 1);
      mbar_init(&bar[B_S + i], 1);
      mbar_init(&bar[B_P + i], 128);
    }
    mbar_init(&bar[B_O], 1);
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

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tmQ);
      tma_prefetch_desc(&tmK);
      tma_prefetch_desc(&tmV);
      mbar_arrive_expect_tx(&bar[B_Q], Cfg::TILE);
      for (int p = 0; p < Cfg::NP; ++p) tma_load_3d(smem + Cfg::OFF_Q + p * Cfg::PANEL, &tmQ, &bar[B_Q], p * 64, head, q0);
      int jj = 0;
      for (int jt = 0; jt < nkt; ++jt) {
        if (tile_kind(a, qpos0, jt) == 0) continue;
        const int st = jj & 1;
        if (jj >= 2) mbar_wait(&bar[B_KVE + st], ((jj - 2) >> 1) & 1);
        uint8_t* sk = smem + Cfg::OFF_K + st * Cfg::TILE;
        uint8_t* sv = smem + Cfg::OFF_V + st * Cfg::TILE;
        mbar_arrive_expect_tx(&bar[B_K + st], Cfg::TILE);
        for (int p = 0; p < Cfg::NP; ++p) tma_load_3d(sk + p * Cfg::PANEL, &tmK, &bar[B_K + st], p * 64, head, jt * WF_TILE);
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
      const uint32_t sQ = smem_u32(smem + Cfg::OFF_Q);
      auto issue_pv = [&](int i) {
        const int st = i & 1;
        mbar_wait(&bar[B_P + st], (i >> 1) & 1);
        mbar_wait(&bar[B_V + st], (i >> 1) & 1);
        tc_fence_after();
        const uint32_t sV = smem_u32(smem + Cfg::OFF_V + st * Cfg::TILE);
#pragma unroll
        for (int k = 0; k < WF_TILE / 16; ++k) {
          const uint64_t bd = smem_desc_sw128(sV + k * 2048, Cfg::PANEL, 1024);
          mma_ts(tbase + 256, tbase + st * 128 + k * 8, bd, idO, (i > 0 || has_state || k > 0) ? 1u : 0u);
        }
        mma_commit(&bar[B_KVE + st]);
        mma_commit(&bar[B_O]);
      };
      mbar_wait(&bar[B_Q], 0);
      tc_fence_after();
      int jj = 0;
      for (int jt = 0; jt < nkt; ++jt) {
        if (tile_kind(a, qpos0, jt) == 0) continue;
        const int st = jj & 1;
        mbar_wait(&bar[B_K + st], (jj >> 1) & 1);
        tc_fence_after();
        const uint32_t sK = smem_u32(smem + Cfg::OFF_K + st * Cfg::TILE);
#pragma unroll
        for (int k = 0; k < DP / 16; ++k) {
          const int p = k >> 2, kk = k & 3;
          const uint64_t ad = smem_desc_sw128(sQ + p * Cfg::PANEL + kk * 32, 16, 1024);
          const uint64_t bd = smem_desc_sw128(sK + p * Cfg::PANEL + kk * 32, 16, 1024);
          mma_ss(tbase + st * 128, ad, bd, idS, k > 0 ? 1u : 0u);
        }
        mma_commit(&bar[B_S + st]);
        if (jj > 0) issue_pv(jj - 1);
        ++jj;
      }
      if (jj > 0) issue_pv(jj - 1);
    }
  } else {
    // ------------------------------------------------------------ softmax + epilogue
    const int wq = warp & 3;
    const int row = wq * 32 + lane;
    const uint32_t tl = tbase + (static_cast<uint32_t>(wq * 32) << 16);
    const int grow = q0 + row;
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
        tmem_st16(tl + 256 + c * 16, r);
      }
      tmem_wait_st();
    }
    int jj = 0;
    for (int jt = 0; jt < nkt; ++jt) {
      const int kind = tile_kind(a, qpos0, jt);
      if (kind == 0) continue;
      const int st = jj & 1;
      mbar_wait(&bar[B_S + st], (jj >> 1) & 1);
      tc_fence_after();
      float s[128];
      {
        uint32_t r0[32], r1[32], r2[32], r3[32];
        tmem_ld32(tl + st * 128 + 0, r0);
        tmem_ld32(tl + st * 128 + 32, r1);
        tmem_ld32(tl + st * 128 + 64, r2);
        tmem_ld32(tl + st * 128 + 96, r3);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          s[i] = __uint_as_float(r0[i]);
          s[32 + i] = __uint_as_float(r1[i]);
          s[64 + i] = __uint_as_float(r2[i]);
          s[96 + i] = __uint_as_float(r3[i]);
        }
      }
      if (kind == 2) {
#pragma unroll
        for (int c = 0; c < 128; ++c)
          if (c > row) s[c] = -INFINITY;
      }
      float mx = s[0];
#pragma unroll
      for (int c = 1; c < 128; ++c) mx = fmaxf(mx, s[c]);
      const float mcand = mx * a.scale_log2;
      const bool need = mcand > m + 8.0f;
      if (__any_sync(0xffffffffu, need)) {
        const float mnew = fmaxf(m, mcand);
        const float alpha = (m == -INFINITY) ? 0.f : fast_exp2(m - mnew);
        if (jj > 0 || has_state) {
          if (jj > 0) {
            mbar_wait(&bar[B_O], (jj - 1) & 1);
            tc_fence_after();
          }
#pragma unroll
          for (int c = 0; c < DP / 16; ++c) {
            uint32_t r[16];
            tmem_ld16(tl + 256 + c * 16, r);
            tmem_wait_ld();
#pragma unroll
            for (int i = 0; i < 16; ++i) r[i] = __float_as_uint(__uint_as_float(r[i]) * alpha);
            tmem_st16(tl + 256 + c * 16, r);
          }
        }
        l *= alpha;
        m = mnew;
      }
      const float mm = (m == -INFINITY) ? 0.f : m;
      float rs = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = fast_exp2(fmaf(s[c * 32 + 2 * i], a.scale_log2, -mm));
          const float p1 = fast_exp2(fmaf(s[c * 32 + 2 * i + 1], a.scale_log2, -mm));
          rs += p0 + p1;
          pk[i] = pack_bf16x2(p0, p1);
        }
        tmem_st16(tl + st * 128 + c * 16, pk);
      }
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&bar[B_P + st]);
      l += rs;
      ++jj;
    }
    // epilogue
    const int ntiles = jj;
    if (ntiles > 0) {
      mbar_wait(&bar[B_O], (ntiles - 1) & 1);
      tc_fence_after();
    }
    const bool have_o = ntiles > 0 || has_state;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    a.lse_out[stat_index(head, grow, a.heads, a.lse_blk)] = l > 0.f ? (m + __log2f(l)) * kLn2 : -INFINITY;
#pragma unroll
    for (int c = 0; c < DP / 16; ++c) {
      uint32_t r[16];
      if (have_o) {
        tmem_ld16(tl + 256 + c * 16, r);
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
  dim3 grid(a.nq / WF_TILE, a.heads);
  wf_block_fwd_kernel<D><<<grid, 192, Cfg::SMEM, s>>>(tq, tk, tv, a);
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
