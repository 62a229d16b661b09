// Micro-probe: cost of one attention softmax tile step (pass 1 row max over
// 128 TMEM columns, pass 2 exp2 + bf16 pack + tcgen05.st of P) for one warpgroup,
// with variants that remove pieces.  clock64 per iteration, 1 CTA per SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2403_19708_b200/csrc/askv_ptx.cuh"
using namespace askv;

template <int MODE>  // 0 full, 1 ex2->fmul, 2 no pass1, 3 ex2 poly, 4 packed (r01), 5 row-in-regs (r01b kernel), 6 = 5 without ex2
__global__ void probe(long long* out, float* sink, int iters) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) tmem_alloc(&slot, 256);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  const uint32_t tmem = slot + ((uint32_t)(warp * 32) << 16);
  float init[32];
  for (int e = 0; e < 32; ++e) init[e] = 0.01f * (lane + e);
  for (int c = 0; c < 4; ++c) tmem_st32(tmem + c * 32, init);
  tmem_wait_st();
  float acc = 0.f, m_acc = 1.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float mx = -INFINITY;
    if (MODE >= 5) {
      uint32_t sr[128];
#pragma unroll
      for (int c = 0; c < 4; ++c)
        tmem_ld32_nowait(tmem + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_wait_ld();
      float a0 = fmaxf(__uint_as_float(sr[0]), __uint_as_float(sr[1]));
      float a1 = fmaxf(__uint_as_float(sr[2]), __uint_as_float(sr[3]));
      float a2 = fmaxf(__uint_as_float(sr[4]), __uint_as_float(sr[5]));
      float a3 = fmaxf(__uint_as_float(sr[6]), __uint_as_float(sr[7]));
#pragma unroll
      for (int e = 8; e < 128; e += 8) {
        a0 = fmax3(a0, __uint_as_float(sr[e + 0]), __uint_as_float(sr[e + 1]));
        a1 = fmax3(a1, __uint_as_float(sr[e + 2]), __uint_as_float(sr[e + 3]));
        a2 = fmax3(a2, __uint_as_float(sr[e + 4]), __uint_as_float(sr[e + 5]));
        a3 = fmax3(a3, __uint_as_float(sr[e + 6]), __uint_as_float(sr[e + 7]));
      }
      mx = fmax3(fmax3(a0, a1, a2), a3, -INFINITY) * 1.44f;
      const float neg_m = -(mx > m_acc ? mx : m_acc);
      const float2 sl2v = make_float2(1.44f, 1.44f), negm2 = make_float2(neg_m, neg_m);
      float2 ls0 = make_float2(0.f, 0.f), ls1 = ls0, ls2 = ls0, ls3 = ls0;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const int k = c * 32 + e;
          const float2 x = ffma2(make_float2(__uint_as_float(sr[k]), __uint_as_float(sr[k + 1])),
                                 sl2v, negm2);
          const int pi = e >> 1;  // pair index in the chunk
          const bool poly = (MODE == 7 && (pi & 3) == 3) || (MODE == 8 && (pi % 8) >= 5);
          const float2 pp = MODE == 6 ? x : poly ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
          switch ((e >> 1) & 3) {
            case 0: ls0 = fadd2(ls0, pp); break;
            case 1: ls1 = fadd2(ls1, pp); break;
            case 2: ls2 = fadd2(ls2, pp); break;
            default: ls3 = fadd2(ls3, pp); break;
          }
          pk[e >> 1] = pack_bf16x2(pp.x, pp.y);
        }
        tmem_st16(tmem + 128 + c * 16, pk);
      }
      tmem_wait_st();
      const float2 la = fadd2(ls0, ls1), lb = fadd2(ls2, ls3);
      acc += (la.x + la.y) + (lb.x + lb.y);
      continue;
    }
    if (MODE == 4) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float sv[32];
        tmem_ld32(tmem + c * 32, sv);
        float m0 = fmax3(sv[0], sv[1], sv[2]), m1 = fmax3(sv[3], sv[4], sv[5]);
#pragma unroll
        for (int e = 6; e < 30; e += 4) {
          m0 = fmax3(m0, sv[e], sv[e + 1]);
          m1 = fmax3(m1, sv[e + 2], sv[e + 3]);
        }
        mx = fmax3(mx, fmax3(m0, m1, sv[30]), sv[31]);
      }
      const float neg_m = -(mx > m_acc ? mx : m_acc);
      const float2 sl2v = make_float2(1.44f, 1.44f), negm2 = make_float2(neg_m, neg_m);
      float2 ls0 = make_float2(0.f, 0.f), ls1 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float sv[32];
        tmem_ld32(tmem + c * 32, sv);
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float2 x = ffma2(make_float2(sv[e], sv[e + 1]), sl2v, negm2);
          float2 pp = make_float2(ex2(x.x), ex2(x.y));
          if ((e >> 1) & 1) ls1 = fadd2(ls1, pp); else ls0 = fadd2(ls0, pp);
          pk[e >> 1] = pack_bf16x2(pp.x, pp.y);
        }
        tmem_st16(tmem + 128 + c * 16, pk);
      }
      tmem_wait_st();
      acc += ls0.x + ls0.y + ls1.x + ls1.y;
      continue;
    }
    mx = -INFINITY;
    if (MODE != 2) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        float sv[32];
        tmem_ld32(tmem + c * 32, sv);
        float m4[4] = {sv[0], sv[1], sv[2], sv[3]};
#pragma unroll
        for (int e = 4; e < 32; ++e) m4[e & 3] = fmaxf(m4[e & 3], sv[e]);
        mx = fmaxf(mx, fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3])));
      }
    }
    const float neg_m = -(mx > m_acc ? mx : m_acc);
    float ls[4] = {0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float sv[32];
      tmem_ld32(tmem + c * 32, sv);
      uint32_t pk[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float x0 = fmaf(sv[e], 1.44f, neg_m), x1 = fmaf(sv[e + 1], 1.44f, neg_m);
        float p0, p1;
        if (MODE == 1) { p0 = x0 * 0.5f; p1 = x1 * 0.5f; }
        else if (MODE == 3) { p0 = ex2_poly(x0); p1 = ex2_poly(x1); }
        else { p0 = ex2(x0); p1 = ex2(x1); }
        ls[(e >> 1) & 3] += p0 + p1;
        pk[e >> 1] = pack_bf16x2(p0, p1);
      }
      tmem_st16(tmem + 128 + c * 16, pk);
    }
    tmem_wait_st();
    acc += ls[0] + ls[1] + ls[2] + ls[3];
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 256); }
}

int main() {
  long long* d; float* sink;
  cudaMalloc(&d, 1024 * 8); cudaMalloc(&sink, 1 << 22);
  const char* names[9] = {"full", "ex2->fmul", "no pass1", "ex2 poly", "packed", "row-in-regs",
                          "row-in-regs, no ex2", "regs, 1/4 poly2", "regs, 3/8 poly2"};
  for (int mode = 0; mode < 9; ++mode)
    for (int wgs : {1, 2}) {
      auto k = mode == 0 ? probe<0> : mode == 1 ? probe<1> : mode == 2 ? probe<2>
               : mode == 3 ? probe<3> : mode == 4 ? probe<4> : mode == 5 ? probe<5>
               : mode == 6 ? probe<6> : mode == 7 ? probe<7> : probe<8>;
      const int iters = 200;
      // wgs warpgroups per SM: run 2 CTAs of 128 threads per SM when wgs == 2
      k<<<148 * wgs, 128>>>(d, sink, iters);
      cudaDeviceSynchronize();
      long long h[296]; cudaMemcpy(h, d, 148 * wgs * 8, cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < 148 * wgs; ++i) mx = h[i] > mx ? h[i] : mx;
      printf("%-10s WG/SM=%d: %.0f cycles per tile step\n", names[mode], wgs, mx / iters);
    }
  return 0;
}
