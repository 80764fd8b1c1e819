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

// mode: 0 SS (A, B in smem), 1 TS (A in TMEM); bg: 0 no background, 1 four warps doing
// tcgen05.ld of 128 columns in a loop, 2 four warps doing tcgen05.st of 64 columns
template <int N>
__global__ void __launch_bounds__(256, 1) mma_rate(int mode, int bg, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // operands: A [128 x 64] bf16 K-major (16 KB), B [N x 64] K-major; contents irrelevant
  for (int i = threadIdx.x; i < (16384 + N * 128) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
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
      const uint32_t idesc = idesc_bf16_f32(128, N, 0, 0);
      const uint32_t sA = smem_u32(smem), sB = sA + 16384;
      uint64_t da[4], db[4];
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        da[kk] = smem_desc_sw128(sA + kk * 32, 16, 1024);
        db[kk] = smem_desc_sw128(sB + kk * 32, 16, 1024);
      }
      unsigned long long g0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
      unsigned long long t0 = clock64();
      if (mode == 0) {
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
  } else if (warp >= 4 && bg) {
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
  const int sm = 16384 + N * 128 + 1024;
  cudaFuncSetAttribute(mma_rate<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm);
  for (int it = 0; it < 3; ++it) mma_rate<N><<<sms, 256, sm>>>(mode, bg, d);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long h[5];
  cudaMemcpy(h, d, 40, cudaMemcpyDeviceToHost);
  printf("N=%d %s bg=%s: issue %.1f cyc/mma, complete %.1f cyc/mma (floor %d), %.1f ns/mma = %.0f MHz, bg iters %llu %s\n",
         N, mode ? "TS" : "SS", bg == 0 ? "none" : (bg == 1 ? "tmem-ld" : "tmem-st"), double(h[0]) / kMmas,
         double(h[1]) / kMmas, 128 * N / 256, double(h[4]) / kMmas, 1e3 * double(h[1]) / double(h[4]), h[2],
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int bg = 0; bg < 3; ++bg)
    for (int mode = 0; mode < 2; ++mode) {
      run<128>(mode, bg, sms);
      run<256>(mode, bg, sms);
    }
  return 0;
}
