// reduce.cu -- HBM-bound kernels around the block kernels:
//   * wf_merge_kernel  : Alg. 1 l.11 ReduceScatter_combine:
//                        L = logsumexp_a lse_a, O = sum_a exp(lse_a - L) O_a over the C
//                        partials of this rank's rows -> bf16 O, fp32 LSE.
//   * wf_dsum_kernel   : D = rowsum(dO o O) (flash-attention backward preprocess; reading c12),
//                        stored with the LSE as the block backward consumes them:
//                        -D / sqrt(d) and -LSE log2(e).
//   * wf_sum_kernel    : the backward team reductions (reading c11): out = sum_j part_j
//                        (fp32 partials -> bf16).
// All are bandwidth kernels: 16-byte vector loads/stores, grid-stride, grid sized from
// the SM count.
#include "common.h"
#include "internal.h"

namespace wf {

namespace {

__device__ __forceinline__ float bf2f(uint16_t b) { return __uint_as_float(static_cast<uint32_t>(b) << 16); }

// One thread = 8 contiguous elements (16 B of bf16) of one (row, head); NP = a.nparts.
template <int NP>
__global__ void wf_merge_kernel(MergeArgs a) {
  const int64_t per_row = a.heads * a.D / 8;  // 8-element groups per token row
  const int64_t total = static_cast<int64_t>(a.rows) * per_row;
  for (int64_t g = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; g < total;
       g += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int row = static_cast<int>(g / per_row);
    const int e0 = static_cast<int>(g % per_row) * 8;
    const int head = e0 / a.D;
    // the partials' loads go out first (independent of the LSE values), so every thread has
    // all its O bytes in flight before the LSE arithmetic
    float4 v[NP][2];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      const float4* src = reinterpret_cast<const float4*>(a.o[j] + static_cast<int64_t>(row) * a.heads * a.D + e0);
      v[j][0] = src[0];
      v[j][1] = src[1];
    }
    float l[NP];
    float L = -INFINITY;
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      l[j] = a.lse[j][static_cast<int64_t>(head) * a.lse_stride[j] + row];
      L = fmaxf(L, l[j]);
    }
    float s = 0.f;
    if (L != -INFINITY) {
#pragma unroll
      for (int j = 0; j < NP; ++j) s += __expf(l[j] - L);
    }
    const float Lf = (L == -INFINITY) ? -INFINITY : L + __logf(s);
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (L != -INFINITY) {
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        if (l[j] != -INFINITY) {  // a partial without keys contributes nothing
          const float w = __expf(l[j] - Lf);
          acc[0] = fmaf(w, v[j][0].x, acc[0]);
          acc[1] = fmaf(w, v[j][0].y, acc[1]);
          acc[2] = fmaf(w, v[j][0].z, acc[2]);
          acc[3] = fmaf(w, v[j][0].w, acc[3]);
          acc[4] = fmaf(w, v[j][1].x, acc[4]);
          acc[5] = fmaf(w, v[j][1].y, acc[5]);
          acc[6] = fmaf(w, v[j][1].z, acc[6]);
          acc[7] = fmaf(w, v[j][1].w, acc[7]);
        }
      }
    }
    uint4 out;
    uint32_t* po = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      __nv_bfloat162 b = __floats2bfloat162_rn(acc[2 * i], acc[2 * i + 1]);
      po[i] = *reinterpret_cast<uint32_t*>(&b);
    }
    *reinterpret_cast<uint4*>(a.out + static_cast<int64_t>(row) * a.heads * a.D + e0) = out;
    if (e0 % a.D == 0) a.lse_out[static_cast<int64_t>(head) * a.rows + row] = Lf;
  }
}

// D[h][row] = sum_d dO[row,h,d] * O[row,h,d]; one 8-lane group per (row, head).
__global__ void wf_dsum_kernel(const __nv_bfloat16* __restrict__ dO, const __nv_bfloat16* __restrict__ O,
                               const float* __restrict__ lse, float* __restrict__ nd, float* __restrict__ nl,
                               int rows, int heads, int D, float scale) {
  const int lanes = 8;
  const uint32_t total = static_cast<uint32_t>(rows) * static_cast<uint32_t>(heads);  // < 2^31 (launch_dsum)
  const int sub = threadIdx.x % lanes;
  for (uint32_t g = (blockIdx.x * blockDim.x + threadIdx.x) / lanes; g < total; g += gridDim.x * blockDim.x / lanes) {
    const int row = static_cast<int>(g / static_cast<uint32_t>(heads));  // 32-bit division: no 64-bit software divide
    const int head = static_cast<int>(g - static_cast<uint32_t>(row) * static_cast<uint32_t>(heads));
    const int64_t base = (static_cast<int64_t>(row) * heads + head) * D;
    const int64_t si = static_cast<int64_t>(head) * rows + row;
    const float x = sub == 0 ? lse[si] : 0.f;  // issued with the dO / O loads, not after the reduction
    float acc = 0.f;
#pragma unroll 2
    for (int e = sub * 8; e < D; e += lanes * 8) {
      const uint4 x = *reinterpret_cast<const uint4*>(dO + base + e);
      const uint4 y = *reinterpret_cast<const uint4*>(O + base + e);
      const uint16_t* hx = reinterpret_cast<const uint16_t*>(&x);
      const uint16_t* hy = reinterpret_cast<const uint16_t*>(&y);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc = fmaf(bf2f(hx[i]), bf2f(hy[i]), acc);
    }
#pragma unroll
    for (int o = lanes / 2; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o, lanes);
    if (sub == 0) {
      // the block backward's statistics, converted once per call for its packed FMAs:
      // -D / sqrt(d) and -LSE log2(e) (-inf kept for query rows without any key)
      nd[si] = -acc * scale;
      nl[si] = x == -INFINITY ? -INFINITY : -x * 1.4426950408889634f;
    }
  }
}

// the same conversion for statistics computed elsewhere (wf_block_bwd's D and LSE)
__global__ void wf_stats_convert_kernel(const float* __restrict__ lse, const float* __restrict__ dsum,
                                        float* __restrict__ nl, float* __restrict__ nd, int64_t n, float scale) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float x = lse[i];
    nl[i] = x == -INFINITY ? -INFINITY : -x * 1.4426950408889634f;
    nd[i] = -dsum[i] * scale;
  }
}

// out[i] = bf16(sum_j part_j[i]), 4 elements per thread.
__global__ void wf_sum_kernel(SumArgs a) {
  const int64_t n4 = a.n / 4;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n4;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int j = 0; j < WF_MAX_PARTS; ++j) {
      if (j < a.nparts) {
        const float4 v = reinterpret_cast<const float4*>(a.parts[j])[i];
        s.x += v.x;
        s.y += v.y;
        s.z += v.z;
        s.w += v.w;
      }
    }
    __nv_bfloat162 lo = __floats2bfloat162_rn(s.x, s.y), hi = __floats2bfloat162_rn(s.z, s.w);
    uint2 o;
    o.x = *reinterpret_cast<uint32_t*>(&lo);
    o.y = *reinterpret_cast<uint32_t*>(&hi);
    reinterpret_cast<uint2*>(a.out)[i] = o;
  }
}

int grid_for(int64_t work, int threads) {
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    if (nsm <= 0) nsm = 148;
  }
  const int64_t blocks = (work + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(nsm) * 8;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

}  // namespace

static_assert(WF_MAX_PARTS == 8, "launch_merge instantiates the merge for 1..8 partials");

cudaError_t launch_merge(const MergeArgs& a, cudaStream_t s) {
  if (a.D % 8 || a.nparts < 1 || a.nparts > WF_MAX_PARTS) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(a.rows) * a.heads * a.D / 8;
  const int g = grid_for(work, 256);
  switch (a.nparts) {
    case 1: wf_merge_kernel<1><<<g, 256, 0, s>>>(a); break;
    case 2: wf_merge_kernel<2><<<g, 256, 0, s>>>(a); break;
    case 3: wf_merge_kernel<3><<<g, 256, 0, s>>>(a); break;
    case 4: wf_merge_kernel<4><<<g, 256, 0, s>>>(a); break;
    case 5: wf_merge_kernel<5><<<g, 256, 0, s>>>(a); break;
    case 6: wf_merge_kernel<6><<<g, 256, 0, s>>>(a); break;
    case 7: wf_merge_kernel<7><<<g, 256, 0, s>>>(a); break;
    default: wf_merge_kernel<8><<<g, 256, 0, s>>>(a); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_dsum(const __nv_bfloat16* dO, const __nv_bfloat16* O, const float* lse, float* nd, float* nl,
                        int rows, int heads, int D, float scale, cudaStream_t s) {
  if (D % 8 || static_cast<int64_t>(rows) * heads >= (int64_t{1} << 31)) return cudaErrorInvalidValue;
  const int64_t work = static_cast<int64_t>(rows) * heads * 8;
  wf_dsum_kernel<<<grid_for(work, 256), 256, 0, s>>>(dO, O, lse, nd, nl, rows, heads, D, scale);
  return cudaGetLastError();
}

cudaError_t launch_stats_convert(const float* lse, const float* dsum, float* nl, float* nd, int64_t n, float scale,
                                 cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  wf_stats_convert_kernel<<<grid_for(n, 256), 256, 0, s>>>(lse, dsum, nl, nd, n, scale);
  return cudaGetLastError();
}

cudaError_t launch_sum(const SumArgs& a, cudaStream_t s) {
  if (a.n % 4 || a.nparts < 1 || a.nparts > WF_MAX_PARTS) return cudaErrorInvalidValue;
  wf_sum_kernel<<<grid_for(a.n / 4, 256), 256, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace wf
