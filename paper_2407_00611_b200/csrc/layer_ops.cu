// layer_ops.cu -- the non-GEMM operators of a WallFacer Transformer layer (SURVEY.md §8(f)
// item 3: the GPT-7B-style block the paper trains): RMSNorm forward/backward,
// SwiGLU forward/backward, the residual add and the packing of (dQ, dK, dV) into one
// [rows, 3E] operand for the projection's backward GEMMs.  All HBM-bound: 16-byte vector
// accesses, one CTA per row for the normalisations (a row is 8 KB at hidden 4096).
#include <cstdint>
#include <cstdio>

#include "../../include/wf.h"
#include "common.h"
#include "internal.h"

namespace wf {
namespace {

using bf16 = __nv_bfloat16;

__device__ __forceinline__ void unpack8(const uint4& v, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 t = __bfloat1622float2(h[i]);
    f[2 * i] = t.x;
    f[2 * i + 1] = t.y;
  }
}
__device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
  uint4 v;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&v);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return v;
}

template <int NT>
__device__ __forceinline__ float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) t += red[i];
  return t;
}

constexpr int kNormThreads = 256;

// y = x * rstd * w, rstd = 1 / sqrt(mean(x^2) + eps)   (one CTA per row)
__global__ void __launch_bounds__(kNormThreads) rmsnorm_fwd_kernel(const bf16* __restrict__ x, const bf16* __restrict__ w,
                                                                   bf16* __restrict__ y, float* __restrict__ rstd,
                                                                   int H, float eps) {
  __shared__ float red[kNormThreads / 32];
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4* yr = reinterpret_cast<uint4*>(y + row * H);
  const int nv = H / 8;
  float ss = 0.f;
  for (int i = threadIdx.x; i < nv; i += kNormThreads) {
    float f[8];
    unpack8(xr[i], f);
#pragma unroll
    for (int k = 0; k < 8; ++k) ss += f[k] * f[k];
  }
  const float r = rsqrtf(block_sum<kNormThreads>(ss, red) / H + eps);
  if (threadIdx.x == 0) rstd[row] = r;
  for (int i = threadIdx.x; i < nv; i += kNormThreads) {
    float f[8], g[8];
    unpack8(xr[i], f);
    unpack8(wr[i], g);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = f[k] * r * g[k];
    yr[i] = pack8(f);
  }
}

// dx = r (w o dy) - x r^3 mean(w o dy o x);  dw += sum_rows dy o x r   (fp32, atomics per CTA)
__global__ void __launch_bounds__(kNormThreads) rmsnorm_bwd_kernel(const bf16* __restrict__ dy, const bf16* __restrict__ x,
                                                                   const bf16* __restrict__ w,
                                                                   const float* __restrict__ rstd,
                                                                   const bf16* __restrict__ dres, bf16* __restrict__ dx,
                                                                   float* __restrict__ dw, int rows, int H,
                                                                   int rows_per_cta) {
  __shared__ float red[kNormThreads / 32];
  const int nv = H / 8;
  // this thread's dw partial: columns 8 i .. 8 i + 7 for i = threadIdx.x + k * kNormThreads
  constexpr int kMaxV = 4;  // H <= 8 * 256 * 4 = 8192
  float acc[kMaxV][8];
#pragma unroll
  for (int v = 0; v < kMaxV; ++v)
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[v][k] = 0.f;
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(rows, r0 + rows_per_cta);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  for (int64_t row = r0; row < r1; ++row) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * H);
    const float r = rstd[row];
    float dot = 0.f;
#pragma unroll
    for (int v = 0; v < kMaxV; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        float f[8], g[8], d[8];
        unpack8(xr[i], f);
        unpack8(wr[i], g);
        unpack8(dyr[i], d);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          dot += g[k] * d[k] * f[k];
          acc[v][k] += d[k] * f[k] * r;
        }
      }
    }
    const float m = block_sum<kNormThreads>(dot, red) / H;
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * H);
    const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + row * H) : nullptr;
#pragma unroll
    for (int v = 0; v < kMaxV; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        float f[8], g[8], d[8], o[8];
        unpack8(xr[i], f);
        unpack8(wr[i], g);
        unpack8(dyr[i], d);
        if (rr) unpack8(rr[i], o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float t = r * g[k] * d[k] - f[k] * r * r * r * m;
          o[k] = rr ? o[k] + t : t;
        }
        dxr[i] = pack8(o);
      }
    }
  }
#pragma unroll
  for (int v = 0; v < kMaxV; ++v) {
    const int i = threadIdx.x + v * kNormThreads;
    if (i < nv)
#pragma unroll
      for (int k = 0; k < 8; ++k) atomicAdd(dw + 8 * i + k, acc[v][k]);
  }
}

__device__ __forceinline__ float sigmoidf_(float g) { return 1.f / (1.f + __expf(-g)); }

// gu = [gate | up] per row ([rows, 2F]); h = silu(gate) * up
__global__ void swiglu_fwd_kernel(const bf16* __restrict__ gu, bf16* __restrict__ h, int64_t rows, int F) {
  const int64_t nv = rows * (F / 8);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nv;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = t / (F / 8), c = t % (F / 8);
    float g[8], u[8], o[8];
    unpack8(reinterpret_cast<const uint4*>(gu + row * 2 * F)[c], g);
    unpack8(reinterpret_cast<const uint4*>(gu + row * 2 * F + F)[c], u);
#pragma unroll
    for (int k = 0; k < 8; ++k) o[k] = g[k] * sigmoidf_(g[k]) * u[k];
    reinterpret_cast<uint4*>(h + row * F)[c] = pack8(o);
  }
}

// dgate = dh * up * silu'(gate), dup = dh * silu(gate); silu'(g) = s (1 + g (1 - s)), s = sigmoid(g)
__global__ void swiglu_bwd_kernel(const bf16* __restrict__ dh, const bf16* __restrict__ gu, bf16* __restrict__ dgu,
                                  int64_t rows, int F) {
  const int64_t nv = rows * (F / 8);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nv;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = t / (F / 8), c = t % (F / 8);
    float g[8], u[8], d[8], dg[8], du[8];
    unpack8(reinterpret_cast<const uint4*>(gu + row * 2 * F)[c], g);
    unpack8(reinterpret_cast<const uint4*>(gu + row * 2 * F + F)[c], u);
    unpack8(reinterpret_cast<const uint4*>(dh + row * F)[c], d);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const float s = sigmoidf_(g[k]);
      du[k] = d[k] * g[k] * s;
      dg[k] = d[k] * u[k] * s * (1.f + g[k] * (1.f - s));
    }
    reinterpret_cast<uint4*>(dgu + row * 2 * F)[c] = pack8(dg);
    reinterpret_cast<uint4*>(dgu + row * 2 * F + F)[c] = pack8(du);
  }
}

__global__ void add_kernel(const bf16* __restrict__ a, const bf16* __restrict__ b, bf16* __restrict__ y, int64_t nv) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float f[8], g[8];
    unpack8(reinterpret_cast<const uint4*>(a)[i], f);
    unpack8(reinterpret_cast<const uint4*>(b)[i], g);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] += g[k];
    reinterpret_cast<uint4*>(y)[i] = pack8(f);
  }
}

// y [rows, 3E] = [a | b | c] row by row
__global__ void pack3_kernel(const bf16* __restrict__ a, const bf16* __restrict__ b, const bf16* __restrict__ c,
                             bf16* __restrict__ y, int64_t rows, int E) {
  const int64_t nv = rows * 3 * (E / 8);
  for (int64_t t = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; t < nv;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = t / (3 * (E / 8)), j = t % (3 * (E / 8));
    const int part = static_cast<int>(j / (E / 8));
    const int64_t cc = j % (E / 8);
    const bf16* src = part == 0 ? a : (part == 1 ? b : c);
    reinterpret_cast<uint4*>(y + row * 3 * E)[j] = reinterpret_cast<const uint4*>(src + row * E)[cc];
  }
}

int grid_elems(int64_t nv) {
  const int64_t g = (nv + 255) / 256;
  return static_cast<int>(g < 148 * 16 ? (g > 0 ? g : 1) : 148 * 16);
}

}  // namespace
}  // namespace wf

using namespace wf;

static wf_status lerr(wf_status s, const char* m) { return wf_set_static_error(s, m); }
static bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }
static wf_status lcheck(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    std::snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    return wf_set_static_error(WF_ERR_CUDA, buf);
  }
  return WF_OK;
}

extern "C" wf_status wf_rmsnorm_fwd(const void* x, const void* w, int64_t rows, int hidden, float eps, void* y,
                                    float* rstd, void* stream) {
  if (!x || !w || !y || !rstd) return lerr(WF_ERR_ARG, "wf_rmsnorm_fwd: null pointer");
  if (!al16(x) || !al16(w) || !al16(y)) return lerr(WF_ERR_ARG, "wf_rmsnorm_fwd: 16-byte alignment");
  if (rows < 0 || hidden <= 0 || hidden % 8) return lerr(WF_ERR_CONFIG, "wf_rmsnorm_fwd: hidden % 8 != 0");
  if (rows == 0) return WF_OK;
  rmsnorm_fwd_kernel<<<static_cast<unsigned>(rows), kNormThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(x), static_cast<const bf16*>(w), static_cast<bf16*>(y), rstd, hidden, eps);
  return lcheck("rmsnorm_fwd");
}

extern "C" wf_status wf_rmsnorm_bwd(const void* dy, const void* x, const void* w, const float* rstd, const void* dres,
                                    int64_t rows, int hidden, void* dx, float* dw, void* stream) {
  if (!dy || !x || !w || !rstd || !dx || !dw) return lerr(WF_ERR_ARG, "wf_rmsnorm_bwd: null pointer");
  if (!al16(dy) || !al16(x) || !al16(w) || !al16(dx) || (dres && !al16(dres)))
    return lerr(WF_ERR_ARG, "wf_rmsnorm_bwd: 16-byte alignment");
  if (rows < 0 || hidden <= 0 || hidden % 8 || hidden > 8 * kNormThreads * 4)
    return lerr(WF_ERR_CONFIG, "wf_rmsnorm_bwd: hidden % 8 != 0 or hidden > 8192");
  if (rows == 0) return WF_OK;
  const int per = static_cast<int>((rows + 148 * 4 - 1) / (148 * 4));
  const unsigned grid = static_cast<unsigned>((rows + per - 1) / per);
  rmsnorm_bwd_kernel<<<grid, kNormThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(dy), static_cast<const bf16*>(x), static_cast<const bf16*>(w), rstd,
      static_cast<const bf16*>(dres), static_cast<bf16*>(dx), dw, static_cast<int>(rows), hidden, per);
  return lcheck("rmsnorm_bwd");
}

extern "C" wf_status wf_swiglu_fwd(const void* gu, int64_t rows, int ffn, void* h, void* stream) {
  if (!gu || !h) return lerr(WF_ERR_ARG, "wf_swiglu_fwd: null pointer");
  if (!al16(gu) || !al16(h) || ffn % 8) return lerr(WF_ERR_CONFIG, "wf_swiglu_fwd: alignment / ffn % 8");
  const int64_t nv = rows * (ffn / 8);
  if (nv == 0) return WF_OK;
  swiglu_fwd_kernel<<<grid_elems(nv), 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const bf16*>(gu),
                                                                                    static_cast<bf16*>(h), rows, ffn);
  return lcheck("swiglu_fwd");
}

extern "C" wf_status wf_swiglu_bwd(const void* dh, const void* gu, int64_t rows, int ffn, void* dgu, void* stream) {
  if (!dh || !gu || !dgu) return lerr(WF_ERR_ARG, "wf_swiglu_bwd: null pointer");
  if (!al16(dh) || !al16(gu) || !al16(dgu) || ffn % 8) return lerr(WF_ERR_CONFIG, "wf_swiglu_bwd: alignment / ffn % 8");
  const int64_t nv = rows * (ffn / 8);
  if (nv == 0) return WF_OK;
  swiglu_bwd_kernel<<<grid_elems(nv), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(dh), static_cast<const bf16*>(gu), static_cast<bf16*>(dgu), rows, ffn);
  return lcheck("swiglu_bwd");
}

extern "C" wf_status wf_add_bf16(const void* a, const void* b, int64_t n, void* y, void* stream) {
  if (!a || !b || !y) return lerr(WF_ERR_ARG, "wf_add_bf16: null pointer");
  if (!al16(a) || !al16(b) || !al16(y) || n % 8) return lerr(WF_ERR_CONFIG, "wf_add_bf16: alignment / n % 8");
  if (n == 0) return WF_OK;
  add_kernel<<<grid_elems(n / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(a), static_cast<const bf16*>(b), static_cast<bf16*>(y), n / 8);
  return lcheck("add");
}

extern "C" wf_status wf_pack3_bf16(const void* a, const void* b, const void* c, int64_t rows, int E, void* y,
                                   void* stream) {
  if (!a || !b || !c || !y) return lerr(WF_ERR_ARG, "wf_pack3_bf16: null pointer");
  if (!al16(a) || !al16(b) || !al16(c) || !al16(y) || E % 8) return lerr(WF_ERR_CONFIG, "wf_pack3_bf16: alignment / E % 8");
  const int64_t nv = rows * 3 * (E / 8);
  if (nv == 0) return WF_OK;
  pack3_kernel<<<grid_elems(nv), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(a), static_cast<const bf16*>(b), static_cast<const bf16*>(c), static_cast<bf16*>(y), rows,
      E);
  return lcheck("pack3");
}
