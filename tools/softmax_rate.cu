// GPU-box microbenchmark: the forward kernel's exponential loop (exps() in attn_fwd.cu: packed
// scale-and-shift FFMA2, two MUFU.EX2, FADD2 row sum, F2FP pack, one tcgen05.st of 16 packed
// columns per 16 pairs, wait::st) run by W warps per SM with S rows held in registers, to
// see whether the TMEM stores or the warp count cap its throughput.  Exponentials per cycle
// per SM; peak 16.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_00611_b200/csrc \
//        tools/softmax_rate.cu -o /tmp/softmax_rate && /tmp/softmax_rate
#include <cstdio>

#include "sm100.cuh"

using namespace wf::sm100;

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

// MMA: an extra warp (the last one) keeps the tensor pipe busy with back-to-back 128x128x16
// SS MMAs into TMEM columns [256, 384) while the softmax warps run
template <int COLS, bool STORE, bool MMA>
__global__ void __launch_bounds__(544, 1) sm_loop(int iters, unsigned long long* cyc, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ volatile int done;
  const int warp = threadIdx.x >> 5;
  const int nsoft = MMA ? (blockDim.x / 32 - 1) : blockDim.x / 32;
  if (threadIdx.x == 0) done = 0;
  if (warp == 0) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (MMA && warp == nsoft) {
    if ((threadIdx.x & 31) == 0) {
      const uint32_t sa = smem_u32(smem), sb = sa + 16384;
      const uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
      unsigned long long n = 0;
      while (!done) {
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)
          mma_ss(tslot + 256, smem_desc_sw128(sa + kk * 32, 16, 1024), smem_desc_sw128(sb + kk * 32, 16, 1024), idesc, 1u);
        ++n;
      }
      if (n == 12345) *sink = 1.f;
    }
    __syncwarp();
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tslot, 512);
    return;
  }
  const uint32_t tl = tslot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + (warp >> 2) * (COLS / 2);
  float s[COLS];
  for (int i = 0; i < COLS; ++i) s[i] = -(threadIdx.x + i) * 1e-3f;
  float tot = 0.f;
  bar_sync_n(2, nsoft * 32);
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float mm = it * 1e-6f;
    const float2 sc2 = make_float2(0.0884f, 0.0884f), nm2 = make_float2(-mm, -mm);
    float2 rs = make_float2(0.f, 0.f);
#pragma unroll
    for (int c = 0; c < COLS / 32; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 x = ffma2(make_float2(s[c * 32 + 2 * i], s[c * 32 + 2 * i + 1]), sc2, nm2);
        const float2 p = make_float2(fast_exp2(x.x), fast_exp2(x.y));
        rs = fadd2(rs, p);
        pk[i] = pack_bf16x2(p.x, p.y);
      }
      if (STORE)
        tmem_st16(tl + c * 16, pk);
      else if (pk[0] == 0x12345u)
        tot += 1.f;
    }
    if (STORE) tmem_wait_st();
    tot += rs.x + rs.y;
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
  if (tot == 1.2345f) *sink = tot;
  if (MMA) {
    bar_sync_n(1, nsoft * 32);
    if (threadIdx.x == 0) done = 1;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tslot, 512);
}

template <int COLS, bool STORE, bool MMA = false>
void run(int warps, int sms) {
  unsigned long long* d;
  float* s;
  cudaMalloc(&d, 8);
  cudaMalloc(&s, 4);
  const int iters = 256;
  cudaFuncSetAttribute(sm_loop<COLS, STORE, MMA>, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  for (int r = 0; r < 2; ++r) sm_loop<COLS, STORE, MMA><<<sms, (warps + (MMA ? 1 : 0)) * 32, 32768 + 1024>>>(iters, d, s);
  cudaError_t e = cudaDeviceSynchronize();
  unsigned long long c;
  cudaMemcpy(&c, d, 8, cudaMemcpyDeviceToHost);
  printf("%3d cols per thread, %2d warps per SM, P stores %s%s: %.2f exponentials/clk/SM %s\n", COLS, warps,
         STORE ? "on " : "off", MMA ? ", tensor pipe busy" : "", double(iters) * COLS * warps * 32 / c, e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(d);
  cudaFree(s);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {4, 8}) {
    run<128, true>(w, sms);
    run<128, false>(w, sms);
  }
  for (int w : {4, 8, 16}) {
    run<64, true>(w, sms);
    run<64, false>(w, sms);
  }
  run<128, true, true>(4, sms);
  run<128, true, true>(8, sms);
  run<64, true, true>(8, sms);
  run<64, true, true>(16, sms);
  return 0;
}
