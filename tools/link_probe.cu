// Probe: pinned-host <-> HBM link throughput for the pre-loader's DMA shapes.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/link_probe tools/link_probe.cu
//   tools/link_probe
//
// Cases: one H2D stream issuing 2.6 MB chunks (a (block, layer) chunk of a
// 13B session) as cudaMemcpyAsync or strided 2-D copies; 2 / 4 concurrent H2D streams;
// H2D with a concurrent D2H stream; 64 MB chunks.  Diagnostics only.
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
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  auto run = [&](const char* name, int nstreams, size_t chunk, bool batch, bool d2h) -> int {
    const size_t n = bytes / chunk;
    for (int rep = 0; rep < 3; ++rep) {
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(a, 0));
      for (int k = 0; k < nstreams; ++k) CK(cudaStreamWaitEvent(st[k], a, 0));
      CK(cudaStreamWaitEvent(sd, a, 0));
      if (d2h) CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, sd));
      for (int k = 0; k < nstreams; ++k) {
        std::vector<void*> ds, ss;
        std::vector<size_t> sz;
        for (size_t i = k; i < n; i += nstreams) {
          ds.push_back(d + i * chunk);
          ss.push_back(h + i * chunk);
          sz.push_back(chunk);
        }
        if (batch) {
          // strided 2-D copies of 23 chunks = one (session, layer) pre-load
          // of consecutive arena blocks (the pre-loader's strided form)
          for (size_t i = 0; i < ds.size(); i += 23) {
            const size_t m = ds.size() - i < 23 ? ds.size() - i : 23;
            const size_t sp = m > 1 ? (size_t)((char*)ss[i + 1] - (char*)ss[i]) : chunk;
            const size_t dp = m > 1 ? (size_t)((char*)ds[i + 1] - (char*)ds[i]) : chunk;
            CK(cudaMemcpy2DAsync(ds[i], dp, ss[i], sp, chunk, m, cudaMemcpyHostToDevice, st[k]));
          }
        } else {
          for (size_t i = 0; i < ds.size(); ++i)
            CK(cudaMemcpyAsync(ds[i], ss[i], chunk, cudaMemcpyHostToDevice, st[k]));
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
    }
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-44s H2D %6.1f GB/s\n", name, (n * chunk) / (ms * 1e-3) / 1e9);
    return 0;
  };
  if (run("1 stream, 2.6 MB memcpy", 1, 2621440, false, false)) return 1;
  if (run("1 stream, 2.6 MB x23 2-D", 1, 2621440, true, false)) return 1;
  if (run("2 streams, 2.6 MB x23 2-D", 2, 2621440, true, false)) return 1;
  if (run("4 streams, 2.6 MB x23 2-D", 4, 2621440, true, false)) return 1;
  if (run("1 stream, 64 MB memcpy", 1, 64 << 20, false, false)) return 1;
  if (run("1 stream, 2.6 MB x23 2-D + 2 GB D2H", 1, 2621440, true, true)) return 1;
  if (run("2 streams, 2.6 MB x23 2-D + 2 GB D2H", 2, 2621440, true, true)) return 1;
  // D2H alone
  {
    CK(cudaDeviceSynchronize());
    CK(cudaEventRecord(a, sd));
    CK(cudaMemcpyAsync(h2, d2, bytes, cudaMemcpyDeviceToHost, sd));
    CK(cudaEventRecord(b, sd));
    CK(cudaEventSynchronize(b));
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("%-44s D2H %6.1f GB/s\n", "1 stream, 2 GB", bytes / (ms * 1e-3) / 1e9);
  }
  return 0;
}
