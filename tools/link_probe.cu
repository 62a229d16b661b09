// Probe: pinned-host <-> HBM link throughput for the pre-loader's / saver's
// DMA shapes (K1 / K4 rooflines).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/link_probe tools/link_probe.cu
//   tools/link_probe
//
// The source is laid out like the host arena: 2.6 MB (block, layer) chunks
// `kStride` chunks apart (a block holds every layer).  Cases: one chunk per
// cudaMemcpyAsync on 1 / 2 / 4 round-robin streams; runs of 23 consecutive
// blocks as one strided cudaMemcpy2DAsync; one 64 MB copy; each with and
// without a concurrent 2 GB D2H; and the concurrent bidirectional pair
// (H2D + D2H rates measured together: the K4 roofline while K1 streams).
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

constexpr size_t kChunk = 2621440;  // 128 tokens x 20 KB (13B row)
constexpr int kStride = 8;          // chunks between consecutive blocks' same layer

int main() {
  const size_t bytes = 2ull << 30;
  char *h, *d, *h2, *d2;
  CK(cudaHostAlloc((void**)&h, bytes, cudaHostAllocDefault));
  CK(cudaHostAlloc((void**)&h2, bytes, cudaHostAllocDefault));
  CK(cudaMalloc((void**)&d, bytes));
  CK(cudaMalloc((void**)&d2, bytes));
  cudaStream_t st[4], sd;
  for (auto& s : st) CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&sd, cudaStreamNonBlocking));
  cudaEvent_t a, b, da, db;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventCreate(&da));
  CK(cudaEventCreate(&db));
  const size_t n = bytes / kChunk;          // chunks moved per pass
  const size_t blocks = n / kStride;        // blocks in the source
  // mode 0: one memcpy per chunk; 1: 2-D runs of 23 blocks; 2: 64 MB copies
  auto run = [&](const char* name, int nstreams, int mode, bool d2h) -> int {
    float best = 0.f, best_d = 0.f;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, 0));
      for (int k = 0; k < nstreams; ++k) CK(cudaStreamWaitEvent(st[k], a, 0));
      CK(cudaStreamWaitEvent(sd, a, 0));
      if (d2h) {
        CK(cudaEventRecord(da, sd));
        CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, sd));
        CK(cudaEventRecord(db, sd));
      }
      size_t moved = 0;
      int rr = 0;
      for (int layer = 0; layer < kStride; ++layer) {  // one pass per layer offset
        if (mode == 2) {
          const size_t big = 64 << 20;
          for (size_t off = 0; off + big <= bytes / kStride; off += big, ++rr) {
            CK(cudaMemcpyAsync(d + layer * (bytes / kStride) + off,
                               h + layer * (bytes / kStride) + off, big,
                               cudaMemcpyHostToDevice, st[rr % nstreams]));
            moved += big;
          }
          continue;
        }
        for (size_t blk = 0; blk < blocks;) {
          const size_t m = mode == 1 ? (blocks - blk < 23 ? blocks - blk : 23) : 1;
          char* dst = d + (layer * blocks + blk) * kChunk;
          const char* src = h + (blk * kStride + layer) * kChunk;
          if (m == 1)
            CK(cudaMemcpyAsync(dst, src, kChunk, cudaMemcpyHostToDevice, st[rr % nstreams]));
          else
            CK(cudaMemcpy2DAsync(dst, kChunk, src, kStride * kChunk, kChunk, m,
                                 cudaMemcpyHostToDevice, st[rr % nstreams]));
          ++rr;
          blk += m;
          moved += m * kChunk;
        }
      }
      for (int k = 0; k < nstreams; ++k) {
        cudaEvent_t ev;
        CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
        CK(cudaEventRecord(ev, st[k]));
        CK(cudaStreamWaitEvent(0, ev, 0));
        cudaEventDestroy(ev);
      }
      CK(cudaEventRecord(b, 0));
      CK(cudaEventSynchronize(b));
      if (d2h) CK(cudaEventSynchronize(db));
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      const float gbs = moved / (ms * 1e-3f) / 1e9f;
      if (gbs > best) best = gbs;
      if (d2h) {
        CK(cudaEventElapsedTime(&ms, da, db));
        const float g2 = bytes / (ms * 1e-3f) / 1e9f;
        if (g2 > best_d) best_d = g2;
      }
    }
    if (d2h)
      printf("%-46s H2D %6.1f GB/s   concurrent D2H %6.1f GB/s\n", name, best, best_d);
    else
      printf("%-46s H2D %6.1f GB/s\n", name, best);
    return 0;
  };
  if (run("1 stream, 2.6 MB chunk per memcpy", 1, 0, false)) return 1;
  if (run("2 streams, 2.6 MB chunk per memcpy", 2, 0, false)) return 1;
  if (run("4 streams, 2.6 MB chunk per memcpy", 4, 0, false)) return 1;
  if (run("1 stream, 23-block 2-D runs", 1, 1, false)) return 1;
  if (run("2 streams, 23-block 2-D runs", 2, 1, false)) return 1;
  if (run("1 stream, 64 MB memcpy", 1, 2, false)) return 1;
  if (run("1 stream, 2.6 MB chunk per memcpy + D2H", 1, 0, true)) return 1;
  if (run("2 streams, 2.6 MB chunk per memcpy + D2H", 2, 0, true)) return 1;
  if (run("1 stream, 23-block 2-D runs + D2H", 1, 1, true)) return 1;
  if (run("1 stream, 64 MB memcpy + D2H", 1, 2, true)) return 1;
  // the saver's shape: D2H of 2 / 6 MB pieces (one layer's new rows of a
  // 100 / 301-token turn) on one stream while a large H2D streams
  for (size_t piece : {(size_t)2 << 20, (size_t)6 << 20}) {
    for (int with_h2d = 0; with_h2d < 2; ++with_h2d) {
      float best = 0.f;
      for (int rep = 0; rep < 3; ++rep) {
        CK(cudaDeviceSynchronize());
        if (with_h2d) CK(cudaMemcpyAsync(d2, h2, bytes, cudaMemcpyHostToDevice, st[1]));
        CK(cudaEventRecord(a, sd));
        size_t moved = 0;
        for (size_t off = 0; off + piece <= bytes / 4; off += piece, moved += piece)
          CK(cudaMemcpyAsync(h + off * 3, d + off, piece, cudaMemcpyDeviceToHost, sd));
        CK(cudaEventRecord(b, sd));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        const float g = moved / (ms * 1e-3f) / 1e9f;
        if (g > best) best = g;
      }
      CK(cudaDeviceSynchronize());
      printf("D2H %zu MB pieces, one stream%-22s D2H %6.1f GB/s\n", piece >> 20,
             with_h2d ? ", 2 GB H2D running" : "", best);
    }
  }
  {
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, sd));
    CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, sd));
    CK(cudaEventRecord(b, sd));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-46s D2H %6.1f GB/s\n", "1 stream, 2 GB D2H alone", bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
