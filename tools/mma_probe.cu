// Micro-probe: raw tcgen05.mma throughput on one SM for the attention tile
// shapes (M=128, N=128, K=16 bf16), SS (A,B in smem) vs TS (A in TMEM),
// measured with clock64 around N back-to-back MMAs + one commit.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2403_19708_b200/csrc/askv_ptx.cuh"
using namespace askv;

template <int MODE>  // 0: SS 128x128, 1: TS 128x128, 2: SS 128x256
__global__ void probe(long long* out, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_mbar_init(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before(); __syncthreads(); tc_fence_after();
  uint32_t tmem = slot;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0x3c003c00u;
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    const int N = MODE == 2 ? 256 : 128;
    const uint32_t idesc = idesc_bf16_f32(128, N, 0, MODE == 1 ? 1 : 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
        if (MODE == 1)
          umma_bf16_tmem_a(tmem + 256, tmem + k * 8, sdesc_sw128(sb + k * 2048, 16384, 1024), idesc, k > 0);
        else
          umma_bf16(tmem, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(sb + off, 16, 1024), idesc, k > 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before(); __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

int main() {
  long long* d; cudaMalloc(&d, 1024 * sizeof(long long));
  long long h[1024];
  const char* names[3] = {"SS 128x128x16", "TS 128x128x16", "SS 128x256x16"};
  for (int mode = 0; mode < 3; ++mode) {
    for (int grid : {1, 148}) {
      auto k = mode == 0 ? probe<0> : mode == 1 ? probe<1> : probe<2>;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
      const int iters = 2000;
      k<<<grid, 128, 100 * 1024>>>(d, iters);
      cudaError_t e = cudaDeviceSynchronize();
      if (e) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
      cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
      double mx = 0; for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
      const int N = mode == 2 ? 256 : 128;
      double macs = 128.0 * N * 16 * 8 * iters;
      printf("%s grid=%d: %.1f cycles/MMA, %.0f MAC/clk/SM\n", names[mode], grid,
             mx / (8.0 * iters), macs / mx);
    }
  }
  return 0;
}
