// layer_ops.cu -- the non-GEMM operators of a WallFacer Transformer layer (SURVEY.md §8(f)
// item 3; "finalized after a standard LayerNorm and FeedForward layer process"):
// LayerNorm forward/backward, the FeedForward layer's GELU forward/backward, the residual
// add and the packing of (dQ, dK, dV) into one [rows, 3E] operand for the projection's
// backward GEMMs.  All HBM-bound: 16-byte vector accesses, one CTA per row for the
// normalisations (a row is 8 KB at hidden 4096).
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
constexpr int kMaxV = 4;  // 16-byte vectors per thread: hidden <= 8 * 256 * 4 = 8192

// LayerNorm (nn.LayerNorm with affine weight and bias; "a standard LayerNorm"):
// y = (x - mean) rstd w + b, rstd = 1 / sqrt(var + eps), var the biased row variance.
// One CTA per row; the row stays in registers between the two reductions.
__global__ void __launch_bounds__(kNormThreads) layernorm_fwd_kernel(const bf16* __restrict__ x,
                                                                     const bf16* __restrict__ w,
                                                                     const bf16* __restrict__ b, bf16* __restrict__ y,
                                                                     float* __restrict__ mean_out,
                                                                     float* __restrict__ rstd_out, int H, float eps) {
  __shared__ float red[kNormThreads / 32];
  const int64_t row = blockIdx.x;
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
  uint4* yr = reinterpret_cast<uint4*>(y + row * H);
  const int nv = H / 8;
  float f[kMaxV][8];
  float s = 0.f;
#pragma unroll
  for (int v = 0; v < kMaxV; ++v) {
    const int i = threadIdx.x + v * kNormThreads;
    if (i < nv) {
      unpack8(xr[i], f[v]);
#pragma unroll
      for (int k = 0; k < 8; ++k) s += f[v][k];
    }
  }
  const float mu = block_sum<kNormThreads>(s, red) / H;
  float ss = 0.f;
#pragma unroll
  for (int v = 0; v < kMaxV; ++v) {
    const int i = threadIdx.x + v * kNormThreads;
    if (i < nv)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const float t = f[v][k] - mu;
        ss += t * t;
      }
  }
  const float r = rsqrtf(block_sum<kNormThreads>(ss, red) / H + eps);
  if (threadIdx.x == 0) {
    mean_out[row] = mu;
    rstd_out[row] = r;
  }
#pragma unroll
  for (int v = 0; v < kMaxV; ++v) {
    const int i = threadIdx.x + v * kNormThreads;
    if (i < nv) {
      float g[8], bb[8], o[8];
      unpack8(reinterpret_cast<const uint4*>(w)[i], g);
      unpack8(reinterpret_cast<const uint4*>(b)[i], bb);
#pragma unroll
      for (int k = 0; k < 8; ++k) o[k] = (f[v][k] - mu) * r * g[k] + bb[k];
      yr[i] = pack8(o);
    }
  }
}

// xhat = (x - mean) rstd, g = w o dy:
//   dx = rstd (g - mean(g) - xhat mean(g o xhat))  (+ dres: the residual branch's gradient)
//   dw += sum_rows dy o xhat,  db += sum_rows dy     (fp32; per-CTA partials, one atomic each)
__global__ void __launch_bounds__(kNormThreads) layernorm_bwd_kernel(
    const bf16* __restrict__ dy, const bf16* __restrict__ x, const bf16* __restrict__ w,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, const bf16* __restrict__ dres,
    bf16* __restrict__ dx, float* __restrict__ dw, float* __restrict__ db, int rows, int H, int rows_per_cta) {
  __shared__ float red[kNormThreads / 32];
  const int nv = H / 8;
  float aw[kMaxV][8], ab[kMaxV][8];
#pragma unroll
  for (int v = 0; v < kMaxV; ++v)
#pragma unroll
    for (int k = 0; k < 8; ++k) aw[v][k] = ab[v][k] = 0.f;
  const int r0 = blockIdx.x * rows_per_cta;
  const int r1 = min(rows, r0 + rows_per_cta);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  for (int64_t row = r0; row < r1; ++row) {
    const uint4* xr = reinterpret_cast<const uint4*>(x + row * H);
    const uint4* dyr = reinterpret_cast<const uint4*>(dy + row * H);
    const float mu = mean_in[row], r = rstd_in[row];
    float xh[kMaxV][8], g[kMaxV][8];
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int v = 0; v < kMaxV; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        float f[8], ww[8], d[8];
        unpack8(xr[i], f);
        unpack8(wr[i], ww);
        unpack8(dyr[i], d);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          xh[v][k] = (f[k] - mu) * r;
          g[v][k] = ww[k] * d[k];
          sg += g[v][k];
          sgx += g[v][k] * xh[v][k];
          aw[v][k] += d[k] * xh[v][k];
          ab[v][k] += d[k];
        }
      }
    }
    const float mg = block_sum<kNormThreads>(sg, red) / H;
    const float mgx = block_sum<kNormThreads>(sgx, red) / H;
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * H);
    const uint4* rr = dres ? reinterpret_cast<const uint4*>(dres + row * H) : nullptr;
#pragma unroll
    for (int v = 0; v < kMaxV; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        float o[8];
        if (rr) unpack8(rr[i], o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float t = r * (g[v][k] - mg - xh[v][k] * mgx);
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
      for (int k = 0; k < 8; ++k) {
        atomicAdd(dw + 8 * i + k, aw[v][k]);
        atomicAdd(db + 8 * i + k, ab[v][k]);
      }
  }
}

// GELU (the FeedForward layer's activation, nn.GELU's exact form): h = u Phi(u),
// Phi(u) = (1 + erf(u / sqrt 2)) / 2;  dh/du = Phi(u) + u phi(u), phi(u) = exp(-u^2/2) / sqrt(2 pi)
__device__ __forceinline__ float gelu_cdf(float u) { return 0.5f * (1.f + erff(u * 0.70710678118654752f)); }

__global__ void gelu_fwd_kernel(const bf16* __restrict__ u, bf16* __restrict__ h, int64_t nv) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(u)[i], f);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = f[k] * gelu_cdf(f[k]);
    reinterpret_cast<uint4*>(h)[i] = pack8(f);
  }
}

__global__ void gelu_bwd_kernel(const bf16* __restrict__ dh, const bf16* __restrict__ u, bf16* __restrict__ du,
                                int64_t nv) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float f[8], d[8];
    unpack8(reinterpret_cast<const uint4*>(u)[i], f);
    unpack8(reinterpret_cast<const uint4*>(dh)[i], d);
#pragma unroll
    for (int k = 0; k < 8; ++k)
      d[k] *= gelu_cdf(f[k]) + f[k] * 0.39894228040143268f * __expf(-0.5f * f[k] * f[k]);
    reinterpret_cast<uint4*>(du)[i] = pack8(d);
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

extern "C" wf_status wf_layernorm_fwd(const void* x, const void* w, const void* b, int64_t rows, int hidden,
                                      float eps, void* y, float* mean, float* rstd, void* stream) {
  if (!x || !w || !b || !y || !mean || !rstd) return lerr(WF_ERR_ARG, "wf_layernorm_fwd: null pointer");
  if (!al16(x) || !al16(w) || !al16(b) || !al16(y)) return lerr(WF_ERR_ARG, "wf_layernorm_fwd: 16-byte alignment");
  if (rows < 0 || hidden <= 0 || hidden % 8 || hidden > 8 * kNormThreads * kMaxV)
    return lerr(WF_ERR_CONFIG, "wf_layernorm_fwd: hidden % 8 != 0 or hidden > 8192");
  if (rows == 0) return WF_OK;
  layernorm_fwd_kernel<<<static_cast<unsigned>(rows), kNormThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(x), static_cast<const bf16*>(w), static_cast<const bf16*>(b), static_cast<bf16*>(y),
      mean, rstd, hidden, eps);
  return lcheck("layernorm_fwd");
}

extern "C" wf_status wf_layernorm_bwd(const void* dy, const void* x, const void* w, const float* mean,
                                      const float* rstd, const void* dres, int64_t rows, int hidden, void* dx,
                                      float* dw, float* db, void* stream) {
  if (!dy || !x || !w || !mean || !rstd || !dx || !dw || !db) return lerr(WF_ERR_ARG, "wf_layernorm_bwd: null pointer");
  if (!al16(dy) || !al16(x) || !al16(w) || !al16(dx) || (dres && !al16(dres)))
    return lerr(WF_ERR_ARG, "wf_layernorm_bwd: 16-byte alignment");
  if (rows < 0 || hidden <= 0 || hidden % 8 || hidden > 8 * kNormThreads * kMaxV)
    return lerr(WF_ERR_CONFIG, "wf_layernorm_bwd: hidden % 8 != 0 or hidden > 8192");
  if (rows == 0) return WF_OK;
  const int per = static_cast<int>((rows + 148 * 4 - 1) / (148 * 4));
  const unsigned grid = static_cast<unsigned>((rows + per - 1) / per);
  layernorm_bwd_kernel<<<grid, kNormThreads, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(dy), static_cast<const bf16*>(x), static_cast<const bf16*>(w), mean, rstd,
      static_cast<const bf16*>(dres), static_cast<bf16*>(dx), dw, db, static_cast<int>(rows), hidden, per);
  return lcheck("layernorm_bwd");
}

extern "C" wf_status wf_gelu_fwd(const void* u, int64_t n, void* h, void* stream) {
  if (!u || !h) return lerr(WF_ERR_ARG, "wf_gelu_fwd: null pointer");
  if (!al16(u) || !al16(h) || n % 8) return lerr(WF_ERR_CONFIG, "wf_gelu_fwd: alignment / n % 8");
  if (n == 0) return WF_OK;
  gelu_fwd_kernel<<<grid_elems(n / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(static_cast<const bf16*>(u),
                                                                                   static_cast<bf16*>(h), n / 8);
  return lcheck("gelu_fwd");
}

extern "C" wf_status wf_gelu_bwd(const void* dh, const void* u, int64_t n, void* du, void* stream) {
  if (!dh || !u || !du) return lerr(WF_ERR_ARG, "wf_gelu_bwd: null pointer");
  if (!al16(dh) || !al16(u) || !al16(du) || n % 8) return lerr(WF_ERR_CONFIG, "wf_gelu_bwd: alignment / n % 8");
  if (n == 0) return WF_OK;
  gelu_bwd_kernel<<<grid_elems(n / 8), 256, 0, static_cast<cudaStream_t>(stream)>>>(
      static_cast<const bf16*>(dh), static_cast<const bf16*>(u), static_cast<bf16*>(du), n / 8);
  return lcheck("gelu_bwd");
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
