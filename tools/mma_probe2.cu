// Micro-probe 2: tcgen05.mma cost per instruction in the attention kernels'
// operand patterns (one SM and all SMs), with and without concurrent shared-
// memory writes (what the TMA K/V fill does to the smem ports).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/mma_probe2 tools/mma_probe2.cu
// Modes (M = 128, K = 16 per instruction, 8 instructions per "tile"):
//   0 SS N=128, A fixed (Q), B walks 3 K tiles       (S = Q K^T, kernel 1)
//   1 SS N=64,  A fixed (Q), B walks 6 half tiles     (S, kernel 2)
//   2 TS N=128, A in TMEM (P), B walks 3 V tiles      (O += P V)
//   3 SS N=256, A fixed, B walks                      (S for a 256-key tile)
//   4 TS N=128 with A = Q in TMEM, B walks K tiles    (S with Q resident in TMEM)
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "../paper_2403_19708_b200/csrc/askv_ptx.cuh"
using namespace askv;

template <int MODE_>
__global__ void probe(long long* out, int iters, int writers, int kmap) {
  constexpr int MODE = MODE_ >= 10 ? MODE_ - 10 : MODE_;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint64_t cbar[6];
  __shared__ uint32_t slot;
  __shared__ volatile int done;
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 6; ++i) mbar_init(&cbar[i], 1);
    fence_mbar_init();
    done = 0;
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  for (int i = threadIdx.x; i < 224 * 1024 / 4; i += blockDim.x)
    ((uint32_t*)smem)[i] = 0x3c003c00u ^ (i * 2654435761u & 0x00ff00ffu);
  fence_proxy_async_smem();
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t sa = smem_u32(smem), sb = smem_u32(smem + 32768);
    constexpr int N = MODE == 1 ? 64 : MODE == 3 ? 256 : 128;
    const uint32_t idesc = idesc_bf16_f32(128, N, 0, MODE == 2 ? 1 : 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
      const uint32_t tile = sb + (it % 3) * 32768 + (MODE == 1 ? (it & 1) * 8192 : 0);
#pragma unroll
      if (MODE >= 5) {
        // the K3 group sequence: PV (A = P in TMEM cols [0, 64), D = O at 256)
        // then S (SS, D = cols [0, 128) -- aliasing P, as in the kernel -- or
        // cols [128, 256) with MODE 6: no alias); MODE 7: PV_a, S_a, PV_b, S_b
        // with two groups (a: S 0 / O 256, b: S 128 / O 384), MODE 8 = 7
        // reordered PV_a, PV_b, S_a, S_b
        // KMAP=1: K3's paired shared-memory map -- Q_a at 0, Q_b at 32 KB,
        // K ring at 64 KB (3 x 32 KB), V ring at 160 KB (2 x 32 KB)
        const uint32_t vt = kmap ? sa + 163840 + (it % 2) * 32768 : sb + (it % 3) * 32768;
        const uint32_t kt = kmap ? sa + 65536 + (it % 3) * 32768 : vt;
        auto pv = [&](uint32_t s_col, uint32_t o_col) {
          const uint32_t idp = idesc_bf16_f32(128, 128, 0, 1);
#pragma unroll
          for (int k = 0; k < 8; ++k)
            umma_bf16_tmem_a(tmem + o_col, tmem + s_col + k * 8,
                             sdesc_sw128(vt + k * 2048, 16384, 1024), idp, true);
        };
        auto ss = [&](uint32_t s_col) {
#pragma unroll
          for (int k = 0; k < 8; ++k) {
            const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
            const uint32_t qa = kmap && s_col ? sa + 32768 : sa;
            umma_bf16(tmem + s_col, sdesc_sw128(qa + off, 16, 1024),
                      sdesc_sw128(kt + off, 16, 1024), idesc, k > 0);
          }
        };
        if (MODE == 9) {  // = 7 with the kernel's commits (o_full, s_full, v_empty, k_empty)
          // KMAP=2: also the kernel's handshake before each group -- a wait
          // on an already completed mbarrier phase + tcgen05.fence::after_thread_sync
          if (kmap == 2) { mbar_wait(&bar, 1); tc_fence_after(); }
          pv(0, 256); umma_commit(&cbar[0]); ss(0); umma_commit(&cbar[1]);
          if (kmap == 2) { mbar_wait(&bar, 1); tc_fence_after(); }
          pv(128, 384); umma_commit(&cbar[2]); ss(128); umma_commit(&cbar[3]);
          umma_commit(&cbar[4]); umma_commit(&cbar[5]);
          continue;
        }
        if (MODE == 5) { pv(0, 256); ss(0); }
        else if (MODE == 6) { pv(0, 256); ss(128); }
        else if (MODE == 7) { pv(0, 256); ss(0); pv(128, 384); ss(128); }
        else { pv(0, 256); pv(128, 384); ss(0); ss(128); }
        continue;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
        if (MODE == 2)
          umma_bf16_tmem_a(tmem + 256, tmem + k * 8, sdesc_sw128(tile + k * 2048, 16384, 1024),
                           idesc, k > 0);
        else if (MODE == 4)
          umma_bf16_tmem_a(tmem + 256, tmem + k * 8, sdesc_sw128(tile + off, 16, 1024), idesc,
                           k > 0);
        else
          umma_bf16(tmem, sdesc_sw128(sa + off, 16, 1024), sdesc_sw128(tile + off, 16, 1024),
                    idesc, k > 0);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    done = 1;
  } else if (warp >= 1 && warp <= writers && MODE_ >= 10) {
    // TMEM reader: tcgen05.ld 32 lanes x 32 columns in a loop over columns
    // [384, 512) (the softmax's S reads), 4 warps cover the 128 lanes
    const uint32_t lane_off = (uint32_t)(((warp - 1) & 3) * 32) << 16;
    float acc = 0.f;
    while (!done) {
#pragma unroll 1
      for (int c = 0; c < 4; ++c) {
        float v[32];
        tmem_ld32(tmem + lane_off + 384 + c * 32, v);
        acc += v[0];
      }
    }
    if (acc == 12345.f) out[0] = 0;
  } else if (warp >= 1 && warp <= writers) {
    // smem writer: 16-byte stores over a 32 KB region (a TMA fill stand-in)
    uint4* w = reinterpret_cast<uint4*>(smem + 131072);
    const uint4 v = make_uint4(1, 2, 3, 4);
    int i = (warp - 1) * 32 + (threadIdx.x & 31);
    while (!done) {
#pragma unroll 8
      for (int r = 0; r < 64; ++r) w[(i + r * 128) & 2047] = v;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * sizeof(long long));
  const int smem = 226 * 1024;
  const char* names[] = {"SS N=128 (S, kernel 1)", "SS N=64 (S, kernel 2)", "TS N=128 (PV)",
                         "SS N=256", "TS N=128 A=Q in TMEM (S)", "PV then S over P (alias)",
                         "PV then S, no alias", "PVa Sa PVb Sb (K3 paired)",
                         "PVa PVb Sa Sb (reordered)", "K3 paired + 6 commits"};
  auto run = [&](auto kern, int mode) {
    if (mode > 9) mode -= 10;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int writers : {0, 4}) {
      for (int grid : {1, 148}) {
        const int iters = getenv("ITERS") ? atoi(getenv("ITERS")) : 400;
        kern<<<grid, 160, smem>>>(d, iters, writers, getenv("KMAP") ? atoi(getenv("KMAP")) : 0);
        cudaError_t e = cudaDeviceSynchronize();
        if (e) {
          printf("err %s\n", cudaGetErrorString(e));
          return;
        }
        long long h[148];
        cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        double mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const int n = mode == 1 ? 64 : mode == 3 ? 256 : 128;
        const double per_it = mode == 5 || mode == 6 ? 16.0 : mode >= 7 ? 32.0 : 8.0;  // 9: 32
        printf("%-26s grid=%3d smem-writers=%d: %6.1f cycles/MMA (%5.0f MAC/clk/SM)\n",
               names[mode], grid, writers, mx / (iters * per_it),
               128.0 * n * 16 * iters * per_it / mx);
      }
    }
  };
  if (getenv("MIX_ONLY")) {
    run(probe<5>, 5);
    run(probe<6>, 6);
    run(probe<7>, 7);
    run(probe<8>, 8);
    run(probe<9>, 9);
    return 0;
  }
  if (!getenv("TMEM_ONLY")) {
    run(probe<0>, 0);
    run(probe<1>, 1);
    run(probe<2>, 2);
    run(probe<3>, 3);
    run(probe<4>, 4);
  }
  printf("-- with 4 warps streaming tcgen05.ld (32x32b.x32) from other TMEM columns --\n");
  run(probe<10>, 0);
  run(probe<12>, 2);
  return 0;
}
