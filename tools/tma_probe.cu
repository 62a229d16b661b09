// Micro-probe: how fast can K/V tiles stream L2 -> shared memory per SM with
// TMA, unicast vs cluster multicast (each CTA of a cluster fetches 1/C of
// every 32 KB tile and multicasts it to all C CTAs)?  Same tensor layout as
// the attention kernel (rows [T][2][H][128] bf16, 3-D map {d, head, row}).
// A consumer warp releases each stage as soon as it lands (no compute), so
// this is the ceiling of the K/V stream alone.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/tma_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "../paper_2403_19708_b200/csrc/askv_ptx.cuh"
using namespace askv;

constexpr int kTile = 32768;   // 128 rows x 128 d x bf16

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::
                   : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(bar)), "r"(cta));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote)
               : "memory");
}
__device__ __forceinline__ void tma_load_mc(void* dst, const void* desc, uint64_t* bar, int c0,
                                            int c1, int c2, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(desc), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
      : "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// grid.x = heads * per_head; CTA (head, q) streams n_tiles K tiles and V tiles.
// kMma: warp 2 keeps the tensor core busy with SS MMAs (M=128 N=128 K=16, both
// operands from a separate 64 KB shared region, like S = Q K^T) while the
// stream runs -- does operand traffic slow the TMA fill?
template <int C, int kStages, int kPieceRows, bool kMma = false>
__global__ void __launch_bounds__(96, 1)
    stream_kernel(const __grid_constant__ CUtensorMap tm, int per_head, int hkv, int n_tiles,
                  int kv_rows) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) &
                                             ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * kTile);
  uint64_t* empty = full + kStages;
  const int head = blockIdx.x / per_head;
  const uint32_t rank = C > 1 ? cluster_rank() : 0;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], C);
    }
    fence_mbar_init();
  }
  __shared__ uint32_t tslot;
  __shared__ volatile int stream_done;
  __shared__ uint64_t mma_bar;
  if (kMma) {
    if (threadIdx.x == 0) {
      stream_done = 0;
      mbar_init(&mma_bar, 1);
      fence_mbar_init();
    }
    if (warp == 2) tmem_alloc(&tslot, 128);
    tc_fence_before();
  }
  if (C > 1) cluster_sync_all(); else __syncthreads();
  if (kMma) tc_fence_after();
  const int steps = 2 * n_tiles;  // K tile, V tile, K tile, ...
  if (warp == 0 && lane == 0) {
    const uint64_t pol = l2_policy_evict_last();
    for (int i = 0; i < steps; ++i) {
      const int s = i % kStages;
      if (i >= kStages) mbar_wait_cluster(&empty[s], ((i / kStages) - 1) & 1);
      mbar_expect_tx(&full[s], kTile);
      const int j = i >> 1, kv = i & 1;
      const int row0 = (j * 128) % kv_rows;
      constexpr int kRH = 128 / kPieceRows, kPieces = 2 * kRH;
      for (int pc = 0; pc < kPieces; ++pc) {
        if (C > 1 && (pc % C) != (int)rank) continue;
        const int dh = pc & 1, rh = pc >> 1;
        uint8_t* dst = smem + s * kTile + dh * 16384 + rh * kPieceRows * 128;
        if (C == 1)
          tma_load_3d_hint(dst, &tm, &full[s], dh * 64, kv * hkv + head % hkv,
                           row0 + rh * kPieceRows, pol);
        else
          tma_load_mc(dst, &tm, &full[s], dh * 64, kv * hkv + head % hkv,
                      row0 + rh * kPieceRows, (uint16_t)((1u << C) - 1));
      }
    }
  } else if (warp == 1 && lane == 0) {
    for (int i = 0; i < steps; ++i) {
      const int s = i % kStages;
      mbar_wait(&full[s], (i / kStages) & 1);
      if (C == 1) {
        mbar_arrive(&empty[s]);
      } else {
        for (int c = 0; c < C; ++c) mbar_arrive_remote(&empty[s], c);
      }
    }
    if (kMma) stream_done = 1;
  } else if (kMma && warp == 2 && lane == 0) {
    const uint32_t sa = smem_u32(smem + kStages * kTile + 2 * kStages * 8 + 1024 - 1024 + 0);
    const uint32_t base = (sa + 1023) & ~1023u;
    const uint32_t sq = base, sk = base + 32768;
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128, 0, 0);
    const uint32_t tmem = tslot;
    int iters = 0;
    while (!stream_done) {
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const uint32_t off = (k >> 2) * 16384 + (k & 3) * 32;
        umma_bf16(tmem, sdesc_sw128(sq + off, 16, 1024), sdesc_sw128(sk + off, 16, 1024), idesc,
                  k > 0);
      }
      umma_commit(&mma_bar);
      mbar_wait(&mma_bar, iters & 1);
      ++iters;
    }
  }
  if (kMma) {
    tc_fence_before();
    __syncwarp();
  }
  if (C > 1) cluster_sync_all();
  if (kMma) {
    __syncthreads();
    if (warp == 2) {
      tc_fence_after();
      tmem_dealloc(tslot, 128);
    }
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  const int hkv = 40, hd = 128, kv_rows = 3200;
  const size_t row_elems = 2ull * hkv * hd;
  void* kv;
  cudaMalloc(&kv, kv_rows * row_elems * 2);
  cudaMemset(kv, 0, kv_rows * row_elems * 2);
  void* flush;
  const size_t flush_bytes = 256ull << 20;
  cudaMalloc(&flush, flush_bytes);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto make = [&](CUtensorMap* tm, int box_rows) {
    cuuint64_t dims[3] = {(cuuint64_t)hd, (cuuint64_t)(2 * hkv), (cuuint64_t)kv_rows};
    cuuint64_t strides[2] = {(cuuint64_t)hd * 2, (cuuint64_t)row_elems * 2};
    cuuint32_t box[3] = {64, 1, (cuuint32_t)box_rows};
    cuuint32_t es[3] = {1, 1, 1};
    return ((EncodeFn)fn)(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, kv, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  };
  CUtensorMap tm64, tm128;
  if (make(&tm64, 64) != CUDA_SUCCESS || make(&tm128, 128) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  const int n_tiles = 25;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  auto run = [&](auto kern, int stages, int piece_rows, int heads, int per_head, int C,
                 bool flush_l2) {
    const int smem = stages * kTile + 2 * stages * 8 + 1024 + 65536 + 1024;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(heads * per_head);
    cfg.blockDim = dim3(96);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const CUtensorMap& tm = piece_rows == 64 ? tm64 : tm128;
    float best = 1e30f;
    for (int rep = 0; rep < 12; ++rep) {
      if (flush_l2) cudaMemsetAsync(flush, rep, flush_bytes);
      cudaEventRecord(e0);
      cudaError_t err = cudaLaunchKernelEx(&cfg, kern, tm, per_head, hkv, n_tiles, kv_rows);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      if (err != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        printf("launch failed: %s\n", cudaGetErrorString(err));
        exit(1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep > 1 && ms < best) best = ms;
    }
    const int ctas = heads * per_head;
    const double per_cta = 2.0 * n_tiles * kTile;
    const double cyc = best * 1e-3 * clk_khz * 1e3;
    printf("stages=%d piece_rows=%3d cluster=%d heads=%2d x %d (%3d CTAs) %s: %7.2f us  "
           "smem-fill %5.1f B/clk/SM  %.2f TB/s into smem\n",
           stages, piece_rows, C, heads, per_head, ctas, flush_l2 ? "cold" : "warm", best * 1e3,
           per_cta / cyc, per_cta * ctas / best / 1e9);
  };
  printf("-- with / without concurrent SS MMAs (M128 N128 K16) on the same SM --\n");
  for (int fl = 1; fl >= 0; --fl) {
    run(stream_kernel<1, 4, 128, false>, 4, 128, 40, 3, 1, fl);
    printf("   + MMA: ");
    run(stream_kernel<1, 4, 128, true>, 4, 128, 40, 3, 1, fl);
  }
  if (getenv("TMA_PROBE_MMA_ONLY")) return 0;
  for (int fl = 1; fl >= 0; --fl) {
    run(stream_kernel<1, 4, 64>, 4, 64, 40, 3, 1, fl);
    run(stream_kernel<1, 4, 128>, 4, 128, 40, 3, 1, fl);
    run(stream_kernel<1, 6, 128>, 6, 128, 40, 3, 1, fl);
    run(stream_kernel<1, 6, 64>, 6, 64, 40, 3, 1, fl);
    run(stream_kernel<1, 2, 128>, 2, 128, 40, 3, 1, fl);
    run(stream_kernel<1, 6, 128>, 6, 128, 10, 12, 1, fl);
    run(stream_kernel<1, 6, 128>, 6, 128, 148, 1, 1, fl);
    run(stream_kernel<2, 4, 128>, 4, 128, 40, 2, 2, fl);
    run(stream_kernel<2, 6, 128>, 6, 128, 40, 2, 2, fl);
    run(stream_kernel<2, 6, 64>, 6, 64, 40, 2, 2, fl);
    run(stream_kernel<4, 6, 64>, 6, 64, 20, 4, 4, fl);
  }
  return 0;
}
