// layer_ops.cu -- the non-GEMM operators of a WallFacer Transformer layer (SURVEY.md §8(f)
// item 3; "finalized after a standard LayerNorm and FeedForward layer process"):
// LayerNorm forward/backward, the FeedForward layer's GELU forward/backward, the residual
// add and the packing of (dQ, dK, dV) into one [rows, 3E] operand for the projection's
// backward GEMMs.  All HBM-bound: 16-byte vector accesses; the normalisations run one CTA
// (256 threads) per row at a time, persistent CTAs walking the rows with the next row's
// loads in flight (a row is 8 KB at hidden 4096).
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
// V = 16-byte vectors per thread (hidden <= 8 * 256 * V).  Persistent CTAs walk the rows;
// the next row's loads are issued before the current row's reductions, and w, b stay in
// registers, so each CTA keeps two rows of reads in flight.
template <int V>
__global__ void __launch_bounds__(kNormThreads) layernorm_fwd_kernel(const bf16* __restrict__ x,
                                                                     const bf16* __restrict__ w,
                                                                     const bf16* __restrict__ b, bf16* __restrict__ y,
                                                                     float* __restrict__ mean_out,
                                                                     float* __restrict__ rstd_out, int64_t rows, int H,
                                                                     float eps) {
  __shared__ float red[kNormThreads / 32];
  const int nv = H / 8;
  float g[V][8], bb[V][8];
  uint4 cur[V];
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int i = threadIdx.x + v * kNormThreads;
    if (i < nv) {
      unpack8(reinterpret_cast<const uint4*>(w)[i], g[v]);
      unpack8(reinterpret_cast<const uint4*>(b)[i], bb[v]);
      if (blockIdx.x < rows) cur[v] = reinterpret_cast<const uint4*>(x + blockIdx.x * static_cast<int64_t>(H))[i];
    }
  }
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t nxt_row = row + gridDim.x;
    uint4 nxt[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv && nxt_row < rows) nxt[v] = reinterpret_cast<const uint4*>(x + nxt_row * H)[i];
    }
    float f[V][8];
    float s = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        unpack8(cur[v], f[v]);
#pragma unroll
        for (int k = 0; k < 8; ++k) s += f[v][k];
      }
    }
    const float mu = block_sum<kNormThreads>(s, red) / H;
    float ss = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
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
    uint4* yr = reinterpret_cast<uint4*>(y + row * H);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        float o[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = (f[v][k] - mu) * r * g[v][k] + bb[v][k];
        yr[i] = pack8(o);
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) cur[v] = nxt[v];
  }
}

// xhat = (x - mean) rstd, g = w o dy:
//   dx = rstd (g - mean(g) - xhat mean(g o xhat))  (+ dres: the residual branch's gradient)
//   dw += sum_rows dy o xhat,  db += sum_rows dy     (fp32; per-CTA partials, one atomic each)
// Persistent CTAs walk the rows (next row's x, dy, dres loads issued before the current
// row's reductions); xhat and g are recomputed from the row's raw vectors in the output pass
// instead of being held, which keeps two CTAs per SM.
template <int V>
__global__ void __launch_bounds__(kNormThreads) layernorm_bwd_kernel(
    const bf16* __restrict__ dy, const bf16* __restrict__ x, const bf16* __restrict__ w,
    const float* __restrict__ mean_in, const float* __restrict__ rstd_in, const bf16* __restrict__ dres,
    bf16* __restrict__ dx, float* __restrict__ dw, float* __restrict__ db, int64_t rows, int H) {
  __shared__ float red[kNormThreads / 32];
  const int nv = H / 8;
  float aw[V][8], ab[V][8], ww[V][8];
  uint4 cx[V], cd[V], cr[V];
  const bool has_res = dres != nullptr;
#pragma unroll
  for (int v = 0; v < V; ++v) {
    const int i = threadIdx.x + v * kNormThreads;
#pragma unroll
    for (int k = 0; k < 8; ++k) aw[v][k] = ab[v][k] = 0.f;
    if (i < nv) {
      unpack8(reinterpret_cast<const uint4*>(w)[i], ww[v]);
      if (blockIdx.x < rows) {
        const int64_t o = blockIdx.x * static_cast<int64_t>(H);
        cx[v] = reinterpret_cast<const uint4*>(x + o)[i];
        cd[v] = reinterpret_cast<const uint4*>(dy + o)[i];
        if (has_res) cr[v] = reinterpret_cast<const uint4*>(dres + o)[i];
      }
    }
  }
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t nxt_row = row + gridDim.x;
    uint4 nx[V], nd[V], nr[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv && nxt_row < rows) {
        nx[v] = reinterpret_cast<const uint4*>(x + nxt_row * H)[i];
        nd[v] = reinterpret_cast<const uint4*>(dy + nxt_row * H)[i];
        if (has_res) nr[v] = reinterpret_cast<const uint4*>(dres + nxt_row * H)[i];
      }
    }
    const float mu = mean_in[row], r = rstd_in[row];
    float sg = 0.f, sgx = 0.f;
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        float f[8], d[8];
        unpack8(cx[v], f);
        unpack8(cd[v], d);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (f[k] - mu) * r, gg = ww[v][k] * d[k];
          sg += gg;
          sgx += gg * xh;
          aw[v][k] += d[k] * xh;
          ab[v][k] += d[k];
        }
      }
    }
    const float mg = block_sum<kNormThreads>(sg, red) / H;
    const float mgx = block_sum<kNormThreads>(sgx, red) / H;
    uint4* dxr = reinterpret_cast<uint4*>(dx + row * H);
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const int i = threadIdx.x + v * kNormThreads;
      if (i < nv) {
        float f[8], d[8], o[8];
        unpack8(cx[v], f);
        unpack8(cd[v], d);
        if (has_res) unpack8(cr[v], o);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const float xh = (f[k] - mu) * r, gg = ww[v][k] * d[k];
          const float t = r * (gg - mg - xh * mgx);
          o[k] = has_res ? o[k] + t : t;
        }
        dxr[i] = pack8(o);
      }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
      cx[v] = nx[v];
      cd[v] = nd[v];
      if (has_res) cr[v] = nr[v];
    }
  }
#pragma unroll
  for (int v = 0; v < V; ++v) {
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
// Phi(u) = (1 + erf(u / sqrt 2)) / 2;  dh/du = Phi(u) + u phi(u), phi(u) = exp(-u^2/2) / sqrt(2 pi).
// erf by Abramowitz & Stegun 7.1.26 (|error| <= 1.5e-7, the accuracy of fp32 erff, far below
// the bf16 output's 2^-9): erf(z) = 1 - t (a1 + t (a2 + t (a3 + t (a4 + t a5)))) exp(-z^2),
// t = 1 / (1 + p z), z >= 0 -- one reciprocal and one exponential on the MUFU pipe, whose
// exp(-z^2) = exp(-u^2 / 2) is also phi's, instead of erff's longer FMA-pipe polynomial.
__device__ __forceinline__ float2 gelu_cdf_pdf(float u) {
  const float z = fabsf(u) * 0.70710678118654752f;
  float t;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(t) : "f"(fmaf(0.3275911f, z, 1.f)));
  const float poly =
      t * fmaf(t, fmaf(t, fmaf(t, fmaf(t, 1.061405429f, -1.453152027f), 1.421413741f), -0.284496736f), 0.254829592f);
  float e;  // exp(-z^2) = 2^(-z^2 log2 e)
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(-z * z * 1.4426950408889634f));
  const float erf_abs = 1.f - poly * e;
  const float cdf = 0.5f + 0.5f * copysignf(erf_abs, u);
  return make_float2(cdf, e * 0.39894228040143268f);
}

__global__ void gelu_fwd_kernel(const bf16* __restrict__ u, bf16* __restrict__ h, int64_t nv) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nv;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float f[8];
    unpack8(reinterpret_cast<const uint4*>(u)[i], f);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = f[k] * gelu_cdf_pdf(f[k]).x;
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
    for (int k = 0; k < 8; ++k) {
      const float2 cp = gelu_cdf_pdf(f[k]);
      d[k] *= cp.x + f[k] * cp.y;
    }
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

// persistent grid for the row kernels: as many CTAs as fit on the SMs at once, at most one per row
template <typename K>
unsigned norm_grid(K kern, int64_t rows) {
  int per_sm = 1, dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kNormThreads, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  const int64_t g = static_cast<int64_t>(nsm) * per_sm;
  return static_cast<unsigned>(rows < g ? rows : g);
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
  const int V = (hidden / 8 + kNormThreads - 1) / kNormThreads;
  auto go = [&](auto kern) {
    const unsigned grid = norm_grid(kern, rows);
    kern<<<grid, kNormThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const bf16*>(x), static_cast<const bf16*>(w), static_cast<const bf16*>(b), static_cast<bf16*>(y),
        mean, rstd, rows, hidden, eps);
  };
  switch (V) {
    case 1: go(layernorm_fwd_kernel<1>); break;
    case 2: go(layernorm_fwd_kernel<2>); break;
    case 3: go(layernorm_fwd_kernel<3>); break;
    default: go(layernorm_fwd_kernel<4>); break;
  }
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
  const int V = (hidden / 8 + kNormThreads - 1) / kNormThreads;
  auto go = [&](auto kern) {
    const unsigned grid = norm_grid(kern, rows);
    kern<<<grid, kNormThreads, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const bf16*>(dy), static_cast<const bf16*>(x), static_cast<const bf16*>(w), mean, rstd,
        static_cast<const bf16*>(dres), static_cast<bf16*>(dx), dw, db, rows, hidden);
  };
  switch (V) {
    case 1: go(layernorm_bwd_kernel<1>); break;
    case 2: go(layernorm_bwd_kernel<2>); break;
    case 3: go(layernorm_bwd_kernel<3>); break;
    default: go(layernorm_bwd_kernel<4>); break;
  }
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
