// GPU-box probe: does tcgen05.mma.kind::f16 accept bf16 A/B with an f16 accumulator
// (instruction-descriptor D format 0), and how does the f16 D land in tensor memory?
// One CTA, M = 128, N = 128, K = 64 (4 MMAs), A/B K-major SW128 in shared memory filled
// with small exact values; prints row 0 of TMEM columns 0..127 as raw words and the fp32
// reference.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2407_00611_b200/csrc \
//        tools/f16acc_probe.cu -o /tmp/f16acc_probe && /tmp/f16acc_probe
#include <cstdio>
#include <cstring>

#include <cuda_fp16.h>

#include "sm100.cuh"

using namespace wf::sm100;

__device__ float aval(int m, int k) { return ((m * 3 + k) % 7 - 3) * 0.25f; }
__device__ float bval(int n, int k) { return ((n * 5 + k) % 5 - 2) * 0.5f; }

__global__ void probe(int f16acc, unsigned* out, float* ref) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // K-major SW128: row r, 16-byte chunk c at (c ^ (r & 7)), 8 rows per 1024 B atom
  for (int i = threadIdx.x; i < 128 * 64; i += blockDim.x) {
    const int r = i / 64, k = i % 64, c = k / 8, e = k % 8;
    const int off = (r >> 3) * 1024 + (r & 7) * 128 + ((c ^ (r & 7)) << 4) + e * 2;
    *reinterpret_cast<__nv_bfloat16*>(smem + off) = __float2bfloat16(aval(r, k));
    *reinterpret_cast<__nv_bfloat16*>(smem + 16384 + off) = __float2bfloat16(bval(r, k));
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    tmem_alloc(&tslot, 256);
    tmem_relinquish();
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = f16acc ? (idesc_bf16_f32(128, 128, 0, 0) & ~(3u << 4)) : idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t sa = smem_u32(smem), sb = sa + 16384;
    for (int kk = 0; kk < 4; ++kk)
      mma_ss(tb, smem_desc_sw128(sa + kk * 32, 16, 1024), smem_desc_sw128(sb + kk * 32, 16, 1024), idesc, kk > 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  if (warp == 0) {  // lanes 0..31 = rows 0..31; columns 0..127
    for (int c = 0; c < 128; c += 32) {
      uint32_t r[32];
      tmem_ld32(tb + c, r);
      tmem_wait_ld();
      if (lane == 0)
        for (int i = 0; i < 32; ++i) out[c + i] = r[i];
    }
    if (lane == 0)
      for (int n = 0; n < 128; ++n) {
        float s = 0.f;
        for (int k = 0; k < 64; ++k) s += __bfloat162float(__float2bfloat16(aval(0, k))) * __bfloat162float(__float2bfloat16(bval(n, k)));
        ref[n] = s;
      }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tb, 256);
}

int main() {
  unsigned* d;
  float* rf;
  cudaMalloc(&d, 128 * 4);
  cudaMalloc(&rf, 128 * 4);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768 + 1024);
  for (int f16 = 0; f16 < 2; ++f16) {
    cudaMemset(d, 0xff, 128 * 4);
    probe<<<1, 128, 32768 + 1024>>>(f16, d, rf);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned h[128];
    float r[128];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(r, rf, sizeof(r), cudaMemcpyDeviceToHost);
    printf("%s accumulator: %s\n", f16 ? "f16" : "f32", e == cudaSuccess ? "ok" : cudaGetErrorString(e));
    for (int n = 0; n < 8; ++n) {
      float asf;
      memcpy(&asf, &h[n], 4);
      const unsigned short lo = h[n] & 0xffff, hi = h[n] >> 16;
      printf("  col %3d: raw %08x  as f32 %10.4f  lo/hi f16 %8.4f %8.4f  ref[%d]=%.4f ref[%d]=%.4f\n", n, h[n], asf,
             __half2float(*reinterpret_cast<const __half*>(&lo)), __half2float(*reinterpret_cast<const __half*>(&hi)),
             n, r[n], 2 * n, r[2 * n]);
    }
  }
  return 0;
}
