// Micro-probe: cycles per 128-element softmax exp pass of one thread row
// (one warp per SMSP, 4 warps per CTA, one CTA per SM), comparing the K3
// loop's fp32 MUFU + polynomial mix with MUFU ex2 on packed bf16 pairs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/exp_probe tools/exp_probe.cu
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include "../paper_2403_19708_b200/csrc/askv_ptx.cuh"
using namespace askv;

__device__ __forceinline__ uint32_t ex2_bf16x2(uint32_t x) {
  uint32_t y;
  asm("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float lo, float hi) {
  uint32_t y;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(hi), "f"(lo));
  return y;
}

__device__ __forceinline__ float2 ex2_poly2_deg2(float2 x) {
  x.x = fmaxf(x.x, -126.0f);
  x.y = fmaxf(x.y, -126.0f);
  const float2 magic = make_float2(12582912.0f, 12582912.0f);
  const float2 t = fadd2(x, magic);
  const float2 j = fadd2(t, make_float2(-12582912.0f, -12582912.0f));
  const float2 f = ffma2(j, make_float2(-1.0f, -1.0f), x);
  float2 p = ffma2(make_float2(0.23842735f, 0.23842735f), f,
                   make_float2(0.70344603f, 0.70344603f));
  p = ffma2(p, f, make_float2(1.0004431f, 1.0004431f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

// POLY: bit k set = pair slot k (of 8) uses the polynomial; DEG 2 or 3
template <int POLY, int DEG>
__global__ void probe_mix(long long* out, uint32_t* sink, int iters) {
  float s[128];
#pragma unroll
  for (int e = 0; e < 128; ++e) s[e] = 0.01f * ((threadIdx.x * 7 + e * 13) & 255) - 1.0f;
  uint32_t acc = 0;
  float lsum = 0.f;
  const float sl2 = 0.12f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float neg_m = -1.0f - it * 1e-6f;
    const float2 sl2v = make_float2(sl2, sl2), negm2 = make_float2(neg_m, neg_m);
    float2 ls0 = make_float2(0.f, 0.f), ls1 = ls0, ls2 = ls0, ls3 = ls0;
#pragma unroll
    for (int e = 0; e < 128; e += 2) {
      const float2 x = ffma2(make_float2(s[e], s[e + 1]), sl2v, negm2);
      const bool poly = (POLY >> ((e >> 1) & 7)) & 1;
      const float2 pp = poly ? (DEG == 2 ? ex2_poly2_deg2(x) : ex2_poly2(x))
                             : make_float2(ex2(x.x), ex2(x.y));
      const uint32_t pk = pack_bf16x2(pp.x, pp.y);
      switch ((e >> 1) & 3) {
        case 0: ls0 = fadd2(ls0, pp); break;
        case 1: ls1 = fadd2(ls1, pp); break;
        case 2: ls2 = fadd2(ls2, pp); break;
        default: ls3 = fadd2(ls3, pp); break;
      }
      acc ^= pk;
    }
    const float2 la = fadd2(ls0, ls1), lb = fadd2(ls2, ls3);
    lsum += (la.x + la.y) + (lb.x + lb.y);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(lsum);
}

template <int POLY, int DEG>
void run_mix(const char* name, int threads) {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 256 * 4);
  const int iters = 200;
  probe_mix<POLY, DEG><<<148, threads>>>(d, sink, iters);
  probe_mix<POLY, DEG><<<148, threads>>>(d, sink, iters);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long s = 0;
  for (long long v : h) s += v;
  printf("%-36s %d warps/SMSP: %6lld cycles per row pass (per warp)\n", name, threads / 128,
         s / 148);
  cudaFree(d);
  cudaFree(sink);
}

template <int MODE>
__global__ void probe(long long* out, uint32_t* sink, int iters) {
  float s[128];
#pragma unroll
  for (int e = 0; e < 128; ++e) s[e] = 0.01f * ((threadIdx.x * 7 + e * 13) & 255) - 1.0f;
  uint32_t acc = 0;
  float lsum = 0.f;
  const float sl2 = 0.12f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const float neg_m = -1.0f - it * 1e-6f;
    const float2 sl2v = make_float2(sl2, sl2), negm2 = make_float2(neg_m, neg_m);
    float2 ls0 = make_float2(0.f, 0.f), ls1 = ls0, ls2 = ls0, ls3 = ls0;
#pragma unroll
    for (int e = 0; e < 128; e += 2) {
      const float2 x = ffma2(make_float2(s[e], s[e + 1]), sl2v, negm2);
      uint32_t pk;
      float2 pp;
      if (MODE == 0) {  // K3 today: 3/4 MUFU f32, 1/4 cubic on FMA
        pp = ((e >> 1) & 3) == 3 ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
        pk = pack_bf16x2(pp.x, pp.y);
      } else if (MODE == 1) {  // all MUFU f32
        pp = make_float2(ex2(x.x), ex2(x.y));
        pk = pack_bf16x2(pp.x, pp.y);
      } else {  // packed bf16 pair through MUFU; exact fp32 unpack for the row sum
        pk = ex2_bf16x2(cvt_bf16x2(x.x, x.y));
        pp = make_float2(__uint_as_float(pk << 16), __uint_as_float(pk & 0xffff0000u));
      }
      switch ((e >> 1) & 3) {
        case 0: ls0 = fadd2(ls0, pp); break;
        case 1: ls1 = fadd2(ls1, pp); break;
        case 2: ls2 = fadd2(ls2, pp); break;
        default: ls3 = fadd2(ls3, pp); break;
      }
      acc ^= pk;
    }
    const float2 la = fadd2(ls0, ls1), lb = fadd2(ls2, ls3);
    lsum += (la.x + la.y) + (lb.x + lb.y);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = (t1 - t0) / iters;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc ^ __float_as_uint(lsum);
}

// accuracy of the packed path against fp32 ex2 rounded to bf16
__global__ void accuracy(float* err) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const float x = -20.0f + 20.0f * i / (gridDim.x * blockDim.x);
  const uint32_t pk = ex2_bf16x2(cvt_bf16x2(x, x));
  const float got = __uint_as_float(pk << 16);
  const float want = exp2f(x);
  err[i] = fabsf(got - want) / want;
}

template <int MODE>
void run(const char* name) {
  long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 148 * 128 * 4);
  const int iters = 200;
  probe<MODE><<<148, 128>>>(d, sink, iters);
  probe<MODE><<<148, 128>>>(d, sink, iters);
  long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  long long s = 0;
  for (long long v : h) s += v;
  printf("%-44s %6lld cycles per 128-element row pass (one warp per SMSP)\n", name, s / 148);
  cudaFree(d);
  cudaFree(sink);
}

int main() {
  run<0>("fp32: 3/4 MUFU ex2 + 1/4 cubic (K3 today)");
  run<1>("fp32: all MUFU ex2");
  run<2>("bf16x2: cvt + MUFU ex2.bf16x2 + fp32 sum");
  for (int t : {128, 256}) {
    run_mix<0x88, 3>("poly 1/4 deg3 (K3 today)", t);
    run_mix<0xAA, 3>("poly 1/2 deg3", t);
    run_mix<0x88, 2>("poly 1/4 deg2", t);
    run_mix<0x92, 2>("poly 3/8 deg2", t);
    run_mix<0xAA, 2>("poly 1/2 deg2", t);
    run_mix<0xDA, 2>("poly 5/8 deg2", t);
  }
  const int n = 1 << 20;
  float* e;
  cudaMalloc(&e, n * 4);
  accuracy<<<n / 256, 256>>>(e);
  static float h[1 << 20];
  cudaMemcpy(h, e, n * 4, cudaMemcpyDeviceToHost);
  double mx = 0, mean = 0;
  for (int i = 0; i < n; ++i) { mx = h[i] > mx ? h[i] : mx; mean += h[i]; }
  printf("ex2.bf16x2(cvt(x)) vs exp2f(x), x in [-20, 0]: max rel err %.4f mean %.5f\n", mx, mean / n);
  return 0;
}
