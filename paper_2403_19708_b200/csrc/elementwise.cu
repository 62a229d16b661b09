// Fused elementwise ops of the LLaMA block around the KV-reuse path (sm_100a).
// Not AttentionStore-specific, but they sit between every pair of GEMMs of the
// prefill step, and torch's generic kernels cost 2-3 launches each:
//   askv_rmsnorm   y = x * rsqrt(mean(x^2) + eps) * w      (fp32 math, bf16 io)
//   askv_silu_mul  a = silu(g) * u for gu = [g | u]         (one pass)
// Both are HBM/latency bound: 16-byte vector loads, one CTA per row (rmsnorm)
// or a grid-stride loop sized to the SM count (silu_mul).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "askv_internal.h"

namespace askv {
namespace {

constexpr int kNormThreads = 256;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One CTA per row; each thread keeps its 16-byte vectors in registers between
// the reduction and the scaled write (cols <= 8 * 8 * 256 = 16384).
template <int VPT>
__global__ void __launch_bounds__(kNormThreads)
    rmsnorm_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                   __nv_bfloat16* __restrict__ y, int cols, float eps,
                   unsigned long long* __restrict__ begin) {
  const int row = blockIdx.x;
  if (begin && row == 0 && threadIdx.x == 0) {  // timeline: start of CTA 0 (runtime.cu)
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    *begin = t;
  }
  const int nvec = cols / 8;
  const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)row * cols);
  const uint4* wr = reinterpret_cast<const uint4*>(w);
  uint4 v[VPT], wv[VPT];
  float ss = 0.f;
  // the weight vectors are loaded up front with x, so the scaled write does
  // not wait a second memory latency after the reduction
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = threadIdx.x + i * kNormThreads;
    wv[i] = idx < nvec ? __ldg(wr + idx) : make_uint4(0, 0, 0, 0);
  }
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = threadIdx.x + i * kNormThreads;
    v[i] = idx < nvec ? xr[idx] : make_uint4(0, 0, 0, 0);
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[i]);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 f = __bfloat1622float2(h[k]);
      ss = fmaf(f.x, f.x, fmaf(f.y, f.y, ss));
    }
  }
  __shared__ float red[kNormThreads / 32];
  ss = warp_sum(ss);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = threadIdx.x < kNormThreads / 32 ? red[threadIdx.x] : 0.f;
    t = warp_sum(t);
    if (threadIdx.x == 0) red[0] = t;
  }
  __syncthreads();
  const float scale = rsqrtf(red[0] / (float)cols + eps);
  uint4* yr = reinterpret_cast<uint4*>(y + (int64_t)row * cols);
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int idx = threadIdx.x + i * kNormThreads;
    if (idx >= nvec) break;
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v[i]);
    const __nv_bfloat162* g = reinterpret_cast<const __nv_bfloat162*>(&wv[i]);
    uint4 o;
    uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float2 a = __bfloat1622float2(h[k]);
      const float2 b = __bfloat1622float2(g[k]);
      __nv_bfloat162 r = __floats2bfloat162_rn(a.x * scale * b.x, a.y * scale * b.y);
      op[k] = *reinterpret_cast<uint32_t*>(&r);
    }
    yr[idx] = o;
  }
}

// grid.y = row, grid.x strides the row's 16-byte vectors with kSiluIlp of
// them in flight per thread (no 64-bit division per vector).
constexpr int kSiluIlp = 4;

__global__ void __launch_bounds__(256)
    silu_mul_kernel(const __nv_bfloat16* __restrict__ gu, __nv_bfloat16* __restrict__ out,
                    int ffn) {
  const int vpr = ffn / 8;
  const int r = blockIdx.y;
  const uint4* gr = reinterpret_cast<const uint4*>(gu + (int64_t)r * 2 * ffn);
  const uint4* ur = gr + vpr;
  uint4* orow = reinterpret_cast<uint4*>(out + (int64_t)r * ffn);
  for (int c0 = blockIdx.x * 256 * kSiluIlp + threadIdx.x; c0 < vpr;
       c0 += gridDim.x * 256 * kSiluIlp) {
    uint4 g[kSiluIlp], u[kSiluIlp];
#pragma unroll
    for (int k = 0; k < kSiluIlp; ++k) {
      const int c = c0 + k * 256;
      if (c < vpr) {
        g[k] = gr[c];
        u[k] = ur[c];
      }
    }
#pragma unroll
    for (int k = 0; k < kSiluIlp; ++k) {
      const int c = c0 + k * 256;
      if (c >= vpr) break;
      const __nv_bfloat162* gh = reinterpret_cast<const __nv_bfloat162*>(&g[k]);
      const __nv_bfloat162* uh = reinterpret_cast<const __nv_bfloat162*>(&u[k]);
      uint4 o;
      uint32_t* op = reinterpret_cast<uint32_t*>(&o);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 a = __bfloat1622float2(gh[e]);
        const float2 b = __bfloat1622float2(uh[e]);
        __nv_bfloat162 r2 = __floats2bfloat162_rn(__fdividef(a.x, 1.f + __expf(-a.x)) * b.x,
                                                  __fdividef(a.y, 1.f + __expf(-a.y)) * b.y);
        op[e] = *reinterpret_cast<uint32_t*>(&r2);
      }
      orow[c] = o;
    }
  }
}

}  // namespace
}  // namespace askv

using namespace askv;

extern "C" int askv_rmsnorm(const void* x, const void* w, void* y, int rows, int cols,
                            float eps, void* stream) {
  clear_error();
  return askv::rmsnorm_stamped(x, w, y, rows, cols, eps, stream, nullptr);
}

int askv::rmsnorm_stamped(const void* x, const void* w, void* y, int rows, int cols, float eps,
                          void* stream, unsigned long long* begin) {
  ASKV_REQUIRE(rows >= 0 && cols > 0 && cols % 8 == 0 && cols <= 8 * 8 * kNormThreads,
               "rmsnorm: cols %d must be a multiple of 8 and <= 16384", cols);
  if (rows == 0) return ASKV_OK;
  ASKV_REQUIRE(x && w && y, "rmsnorm: null pointer");
  const int nvec = cols / 8;
  const int vpt = (nvec + kNormThreads - 1) / kNormThreads;
  auto* xi = static_cast<const __nv_bfloat16*>(x);
  auto* wi = static_cast<const __nv_bfloat16*>(w);
  auto* yo = static_cast<__nv_bfloat16*>(y);
  cudaStream_t s = (cudaStream_t)stream;
  switch (vpt) {
    case 1: rmsnorm_kernel<1><<<rows, kNormThreads, 0, s>>>(xi, wi, yo, cols, eps, begin); break;
    case 2: rmsnorm_kernel<2><<<rows, kNormThreads, 0, s>>>(xi, wi, yo, cols, eps, begin); break;
    case 3: rmsnorm_kernel<3><<<rows, kNormThreads, 0, s>>>(xi, wi, yo, cols, eps, begin); break;
    case 4: rmsnorm_kernel<4><<<rows, kNormThreads, 0, s>>>(xi, wi, yo, cols, eps, begin); break;
    default: rmsnorm_kernel<8><<<rows, kNormThreads, 0, s>>>(xi, wi, yo, cols, eps, begin); break;
  }
  return launch_status("rmsnorm launch");
}

extern "C" int askv_silu_mul(const void* gu, void* out, int rows, int ffn, void* stream) {
  clear_error();
  ASKV_REQUIRE(rows >= 0 && ffn > 0 && ffn % 8 == 0, "silu_mul: ffn %d must be a multiple of 8",
               ffn);
  if (rows == 0) return ASKV_OK;
  ASKV_REQUIRE(gu && out, "silu_mul: null pointer");
  ASKV_REQUIRE(rows <= 65535, "silu_mul: %d rows exceed the grid's y limit", rows);
  const int vpr = ffn / 8;
  const dim3 grid((vpr + 256 * kSiluIlp - 1) / (256 * kSiluIlp), rows);
  silu_mul_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(
      static_cast<const __nv_bfloat16*>(gu), static_cast<__nv_bfloat16*>(out), ffn);
  return launch_status("silu_mul launch");
}
