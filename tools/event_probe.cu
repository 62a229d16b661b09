// Probe: what an in-stream event record / cross-stream wait costs on the GPU,
// with and without a saturating pinned-host -> HBM copy on another stream.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/event_probe tools/event_probe.cu
//   tools/event_probe
//
// Each case runs 2000 short kernels (~4 us) back to back on one stream with
// one extra operation between consecutive kernels and reports the per-kernel
// time.  Diagnostics only.
#include <cuda_runtime.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <thread>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e = (x);                                                        \
    if (e != cudaSuccess) {                                                     \
      printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void spin(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

__global__ void stamp(unsigned long long* out, int i) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  out[i] = t;
}

int main() {
  const int N = 2000;
  cudaStream_t s, bg;
  CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&bg, cudaStreamNonBlocking));
  const size_t bytes = 1ull << 30;
  void *h, *d;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocDefault));
  CK(cudaMalloc(&d, bytes));
  unsigned long long* st;
  CK(cudaMalloc(&st, N * sizeof(unsigned long long)));
  cudaEvent_t ev_t[N], ev_n[N], done, a, b;
  for (int i = 0; i < N; ++i) {
    CK(cudaEventCreate(&ev_t[i]));
    CK(cudaEventCreateWithFlags(&ev_n[i], cudaEventDisableTiming));
  }
  CK(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventRecord(done, bg));
  CK(cudaStreamSynchronize(bg));

  std::atomic<bool> stop{false};
  const char* names[] = {"none", "timing event", "no-timing event", "wait done event",
                         "stamp kernel", "graph: timing event", "graph: none",
                         "graph: stamp kernel"};
  for (int busy = 0; busy < 2; ++busy) {
    std::thread t;
    stop = false;
    if (busy) {
      t = std::thread([&] {
        cudaSetDevice(0);
        while (!stop) {
          cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, bg);
          cudaStreamSynchronize(bg);
        }
      });
      std::this_thread::sleep_for(std::chrono::milliseconds(200));
    }
    for (int mode = 0; mode < 8; ++mode) {
      cudaGraphExec_t ge = nullptr;
      auto issue = [&](bool ext) {
        for (int i = 0; i < N; ++i) {
          spin<<<1, 32, 0, s>>>(4000);
          if (mode == 1 || mode == 5)
            cudaEventRecordWithFlags(ev_t[i], s, ext ? cudaEventRecordExternal : 0);
          if (mode == 2) cudaEventRecord(ev_n[i], s);
          if (mode == 3) cudaStreamWaitEvent(s, done, 0);
          if (mode == 4 || mode == 7) stamp<<<1, 1, 0, s>>>(st, i);
        }
      };
      if (mode >= 5) {
        cudaGraph_t g;
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
        issue(true);
        CK(cudaStreamEndCapture(s, &g));
        CK(cudaGraphInstantiate(&ge, g, 0));
        cudaGraphDestroy(g);
      }
      for (int rep = 0; rep < 2; ++rep) {
        CK(cudaStreamSynchronize(s));
        CK(cudaEventRecord(a, s));
        if (ge)
          CK(cudaGraphLaunch(ge, s));
        else
          issue(false);
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
      }
      float ms;
      CK(cudaEventElapsedTime(&ms, a, b));
      printf("%-10s %-22s %7.2f us per kernel\n", busy ? "h2d-busy" : "idle-link", names[mode],
             ms * 1e3f / N);
      if (ge) cudaGraphExecDestroy(ge);
    }
    if (busy) {
      stop = true;
      t.join();
    }
  }
  // copy stream: 1 GiB H2D as 400 chunks of 2.6 MB, with an event per chunk
  for (int mode = 0; mode < 4; ++mode) {
    const size_t chunk = bytes / 400;
    for (int rep = 0; rep < 2; ++rep) {
      CK(cudaStreamSynchronize(bg));
      CK(cudaEventRecord(a, bg));
      for (int i = 0; i < 400; ++i) {
        CK(cudaMemcpyAsync((char*)d + i * chunk, (char*)h + i * chunk, chunk,
                           cudaMemcpyHostToDevice, bg));
        if (mode == 1) CK(cudaEventRecord(ev_t[i], bg));
        if (mode == 2) CK(cudaEventRecord(ev_n[i], bg));
        if (mode == 3) stamp<<<1, 1, 0, bg>>>(st, i);
      }
      CK(cudaEventRecord(b, bg));
      CK(cudaEventSynchronize(b));
    }
    float ms;
    CK(cudaEventElapsedTime(&ms, a, b));
    printf("copy stream, event per 2.6 MB chunk: %-16s %6.1f GB/s\n",
           mode == 0 ? "none" : mode == 1 ? "timing event" : mode == 2 ? "no-timing event"
                                                                       : "stamp kernel",
           400.0 * (bytes / 400) / (ms * 1e-3) / 1e9);
  }
  // globaltimer granularity: distinct consecutive stamp values
  {
    unsigned long long hs[N];
    CK(cudaMemcpy(hs, st, sizeof(hs), cudaMemcpyDeviceToHost));
    unsigned long long mind = ~0ull;
    for (int i = 1; i < 400; ++i)
      if (hs[i] > hs[i - 1] && hs[i] - hs[i - 1] < mind) mind = hs[i] - hs[i - 1];
    printf("smallest positive stamp step over the copy-stream stamps: %llu ns\n", mind);
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed));
    for (int i = 0; i < 200; ++i) stamp<<<1, 1, 0, s>>>(st, i);
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(hs, st, 200 * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    printf("graph of 200 stamp kernels: deltas");
    for (int i = 1; i < 12; ++i) printf(" %llu", hs[i] - hs[i - 1]);
    printf(" ns; total %llu ns\n", hs[199] - hs[0]);
  }
  return 0;
}
