// GPU-box microbenchmark: cycles per tcgen05.mma (kind::f16, bf16 -> fp32) issued back to
// back by one thread with operands resident in shared / tensor memory, for the shapes the
// block kernels use (128 x N x 16, SS and TS forms), alone and with other warps loading or
// storing tensor memory at the same time.  One CTA per SM on every SM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_00611_b200/csrc \
//        tools/mma_rate.cu -o gpurun_out/mma_rate -lcuda && gpurun_out/mma_rate
#include <cstdio>
#include <cstdlib>

#include "sm100.cuh"

using namespace wf::sm100;

constexpr int kMmas = 4096;

// Two groups of 8 MMAs per round, kMmas in total.  TS1/TS2: form of each group; D1/D2:
// accumulator columns; CM: commit after each group; Z: the first MMA of a group overwrites
// (accumulate = 0), as in the block kernels; AB: the second group reads its shared-memory
// operands 16 KB further (another ring stage).
template <bool TS1, bool TS2, int D1, int D2, bool CM, bool Z, bool AB>
__device__ __forceinline__ void groups(uint32_t tbase, const uint64_t (&da)[4], const uint64_t (&db)[4], uint32_t idesc,
                                       uint64_t* cbar) {
  constexpr uint64_t sh = AB ? (16384u >> 4) : 0u;
  for (int i = 0; i < kMmas; i += 16) {
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t acc = (Z && kk == 0) ? 0u : 1u;
      if (TS1)
        mma_ts(tbase + D1, tbase + 384 + (kk & 3) * 8, db[kk & 3], idesc, acc);
      else
        mma_ss(tbase + D1, da[kk & 3], db[kk & 3], idesc, acc);
    }
    if (CM) mma_commit(cbar);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t acc = (Z && kk == 0) ? 0u : 1u;
      if (TS2)
        mma_ts(tbase + D2, tbase + 384 + (kk & 3) * 8, db[kk & 3] + sh, idesc, acc);
      else
        mma_ss(tbase + D2, da[kk & 3] + sh, db[kk & 3] + sh, idesc, acc);
    }
    if (CM) mma_commit(cbar);
  }
}

// mode: 0 SS (A, B in smem), 1 TS (A in TMEM); bg: 0 no background, 1 four warps doing
// tcgen05.ld of 128 columns in a loop, 2 four warps doing tcgen05.st of 64 columns
template <int N>
__global__ void __launch_bounds__(256, 1) mma_rate(int mode, int bg, unsigned long long* out, const uint8_t* gsrc) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar, tbar, cbar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // operands: A [128 x 64] bf16 K-major (16 KB), B [N x 64] K-major; contents irrelevant
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    mbar_init(&tbar, 1);
    mbar_init(&cbar, 1);
    done = 0;
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = tslot;
  if (warp == 0) {
    if (lane == 0) {
      const int a_mn = mode < 8 ? (mode >> 2) & 1 : 0, b_mn = mode < 8 ? (mode >> 1) & 1 : 0;
      const uint32_t idesc = idesc_bf16_f32(128, N, a_mn, b_mn);
      const uint32_t sA = smem_u32(smem), sB = sA + 16384;
      uint64_t da[4], db[4];
      // K-major: k-step kk at +32 B in the 128-B rows; MN-major: 16 K-rows of 128 B = +2048 B,
      // 64-element MN panels LBO = 8 KB (A: 128 rows = 2 panels, B: N / 64 panels) apart
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        da[kk] = a_mn ? smem_desc_sw128(sA + kk * 2048, 8192, 1024) : smem_desc_sw128(sA + kk * 32, 16, 1024);
        db[kk] = b_mn ? smem_desc_sw128(sB + kk * 2048, 8192, 1024) : smem_desc_sw128(sB + kk * 32, 16, 1024);
      }
      unsigned long long g0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
      unsigned long long t0 = clock64();
      if (mode >= 8) {
        // groups of 8 MMAs (one K = 128 contraction each), two groups per round; see groups()
        switch (mode) {
          case 8: groups<false, true, 0, 256, false, false, false>(tbase, da, db, idesc, &cbar); break;
          case 9: groups<false, true, 0, 256, true, false, false>(tbase, da, db, idesc, &cbar); break;
          case 10: groups<false, false, 0, 0, true, false, false>(tbase, da, db, idesc, &cbar); break;
          case 11: groups<false, false, 0, 256, false, false, false>(tbase, da, db, idesc, &cbar); break;
          case 12: groups<false, false, 0, 0, false, true, false>(tbase, da, db, idesc, &cbar); break;
          case 13: groups<false, false, 0, 0, false, false, true>(tbase, da, db, idesc, &cbar); break;
          case 14: groups<true, true, 0, 256, true, false, false>(tbase, da, db, idesc, &cbar); break;
          case 15: groups<false, false, 0, 256, true, true, false>(tbase, da, db, idesc, &cbar); break;
          case 16: groups<false, true, 0, 256, true, true, false>(tbase, da, db, idesc, &cbar); break;
          default: break;
        }
      } else if ((mode & 1) == 0) {
        for (int i = 0; i < kMmas; i += 4)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_ss(tbase, da[kk], db[kk], idesc, 1u);
      } else {
        for (int i = 0; i < kMmas; i += 4)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) mma_ts(tbase, tbase + 256 + kk * 8, db[kk], idesc, 1u);
      }
      unsigned long long t1 = clock64();
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      unsigned long long t2 = clock64(), g2;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g2));
      if (blockIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t2 - t0;
        out[4] = g2 - g0;
      }
      done = 1;
    }
  } else if (warp == 1 && bg == 3) {
    // TMA (bulk copy) loads of 32 KB from a 1 GB buffer into a 64 KB region behind the
    // operands, back to back, as the block kernels' K/V producers do
    if (lane == 0) {
      uint8_t* dst = smem + 16384 + N * 128 + 1024;
      unsigned long long n = 0;
      const size_t span = (size_t(1) << 30) / 32768;
      while (!done) {
        mbar_arrive_expect_tx(&tbar, 32768);
        const uint8_t* src = gsrc + ((blockIdx.x * 977 + n * 148) % span) * 32768;
        for (int c = 0; c < 4; ++c) bulk_load(dst + (n & 1) * 32768 + c * 8192, src + c * 8192, 8192, &tbar);
        mbar_wait(&tbar, n & 1);
        ++n;
      }
      if (blockIdx.x == 0) out[2] = n;
    }
  } else if (warp >= 2 && bg == 4) {
    // six warps of softmax-like work: packed FMAs, exponentials, bf16 packs (ALU/FMA/MUFU)
    float2 x = make_float2(threadIdx.x * 1e-3f, -threadIdx.x * 1e-3f);
    uint32_t acc = 0;
    unsigned long long n = 0;
    while (!done) {
#pragma unroll 16
      for (int i = 0; i < 64; ++i) {
        const float2 y = ffma2(x, make_float2(0.999f, 0.999f), make_float2(-1e-4f, 1e-4f));
        const float2 p = make_float2(fast_exp2(y.x), fast_exp2(y.y));
        acc ^= pack_bf16x2(p.x, p.y);
        x = fadd2(y, make_float2(p.x * 1e-6f, p.y * 1e-6f));
      }
      ++n;
    }
    if (acc == 0x12345u) out[3] = n;
    if (blockIdx.x == 0 && lane == 0 && warp == 4) out[2] = n;
  } else if (warp >= 4 && bg && bg < 3) {
    const uint32_t tl = tbase + (static_cast<uint32_t>((warp & 3) * 32) << 16);
    unsigned long long n = 0;
    while (!done) {
      if (bg == 1) {
        uint32_t r[32];
        tmem_ld32(tl + 384, r);
        tmem_ld32(tl + 416, r);
        tmem_ld32(tl + 448, r);
        tmem_ld32(tl + 480, r);
        tmem_wait_ld();
        if (r[0] == 12345u) out[3] = r[1];
      } else {
        uint32_t r[16];
        for (int i = 0; i < 16; ++i) r[i] = i;
        tmem_st16(tl + 384, r);
        tmem_st16(tl + 400, r);
        tmem_st16(tl + 416, r);
        tmem_st16(tl + 432, r);
        tmem_wait_st();
      }
      ++n;
    }
    if (blockIdx.x == 0 && lane == 0 && warp == 4) out[2] = n;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tbase, 512);
}

template <int N>
void run(int mode, int bg, int sms) {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  const int sm = 16384 + N * 128 + 1024 + 65536;  // operands, barriers, TMA region (+16 KB stage shift fits)
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  static uint8_t* g = nullptr;
  if (!g) cudaMalloc(&g, size_t(1) << 30);
  for (int it = 0; it < 3; ++it) mma_rate<N><<<sms, 256, sm>>>(mode, bg, d, g);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[5];
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("N=%d mode %2d %s%s%s bg=%s: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d), %.1f ns/mma = %.0f MHz, bg iters %llu %s\n",
 N, mode, mode >= 8 ? "groups" : ((mode & 1) ? "TS" : "SS"), (mode < 8 && (mode & 4)) ? " A-MN" : "",
         (mode < 8 && (mode & 2)) ? " B-MN" : "", bg == 0 ? "none" : (bg == 1 ? "tmem-ld" : (bg == 2 ? "tmem-st" : (bg == 3 ? "tma-load" : "softmax-like"))), double(h[0]) / kMmas,
         double(h[1]) / kMmas, 128 * N / 256, double(h[4]) / kMmas, 1e3 * double(h[1]) / double(h[4]), h[2],
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main_pair();

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int modes[] = {0, 1, 2, 3, 4, 6};
  for (int bg = 0; bg < 4; bg += 3)
    for (int mode : modes) {
      run<128>(mode, bg, sms);
      run<256>(mode, bg, sms);
    }
  for (int mode = 8; mode < 17; ++mode) run<128>(mode, 0, sms);
  for (int mode : modes) run<64>(mode, 0, sms);  // N = 64 (the 64-key sub-tile S)
  for (int mode : {0, 1}) {  // with softmax-like compute on six other warps
    run<128>(mode, 4, sms);
    run<64>(mode, 4, sms);
  }
  for (int mode = 8; mode < 10; ++mode) run<128>(mode, 4, sms);
  main_pair();
  return 0;
}

// ---------------------------------------------------------------- CTA-pair (cta_group::2)
// The even CTA of a cluster of two issues M = 256 MMAs (A rows from both CTAs' shared
// memory, B split along N: each CTA holds N / 2 rows), SS or TS (A from both CTAs' TMEM).
__device__ __forceinline__ void mma2_ts_rate(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                             uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

template <int N, bool TS>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2_rate(unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t cr = cluster_ctarank();
  for (int i = threadIdx.x; i < (16384 + N / 2 * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc2(&tslot, 512);
    tmem_relinquish2();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (cr == 0 && warp == 0 && lane == 0) {
    const uint32_t idesc = idesc_bf16_f32(256, N, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    uint64_t da[4], db[4];
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      da[kk] = smem_desc_sw128(sa + kk * 32, 16, 1024);
      db[kk] = smem_desc_sw128(sb + kk * 32, 16, 1024);
    }
    unsigned long long t0 = clock64();
    for (int i = 0; i < kMmas; i += 4)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        if (TS)
          mma2_ts_rate(tb, tb + 256 + kk * 8, db[kk], idesc, 1u);
        else
          mma2_ss(tb, da[kk], db[kk], idesc, 1u);
      }
    unsigned long long t1 = clock64();
    mma2_commit_mc(&bar, 0x3);
    mbar_wait(&bar, 0);
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  } else if (cr == 1 && threadIdx.x == 0) {
    mbar_wait(&bar, 0);  // the multicast commit
  }
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) tmem_dealloc2(tb, 512);
}

template <int N, bool TS>
void run2(int sms) {
  unsigned long long* d;
  cudaMalloc(&d, 64);
  cudaMemset(d, 0, 64);
  const int sm = 16384 + N / 2 * 128 + 1024;
  cudaFuncSetAttribute(mma2_rate<N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  for (int it = 0; it < 3; ++it) mma2_rate<N, TS><<<sms, 128, sm>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("pair M=256 N=%d %s: issue %.1f cyc/mma, complete %.1f cyc/mma (floor per SM %d) %s\n", N, TS ? "TS" : "SS",
         double(h[0]) / kMmas, double(h[1]) / kMmas, 256 * N / 512, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main_pair() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  sms &= ~1;
  run2<128, false>(sms);
  run2<128, true>(sms);
  run2<256, false>(sms);
  run2<256, true>(sms);
  return 0;
}
