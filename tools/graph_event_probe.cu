// Probe: does cudaStreamWaitEvent on another stream, issued after
// cudaGraphLaunch, wait for an external event-record node inside that graph?
// (the native layer loop records ev_save_ready / ev_src_free that way and the
// saver / pre-loader streams wait on them after the launch).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/graph_event_probe tools/graph_event_probe.cu
#include <cuda_runtime.h>

#include <cstdio>

__global__ void spin_then_write(int* flag, int value, unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
  *(volatile int*)flag = value;
}
__global__ void read_flag(const int* flag, int* out) { *out = *(volatile const int*)flag; }

int main() {
  int *flag, *out;
  cudaMalloc(&flag, 4);
  cudaMallocHost(&out, 4);
  cudaStream_t s, s2;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t ev;
  cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  int bad = 0;
  for (int trial = 0; trial < 20; ++trial) {
    cudaMemset(flag, 0, 4);
    cudaDeviceSynchronize();
    // graph: spin 200 us, write flag = trial + 1, external record of ev
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeRelaxed);
    spin_then_write<<<1, 1, 0, s>>>(flag, trial + 1, 200000);
    cudaEventRecordWithFlags(ev, s, cudaEventRecordExternal);
    spin_then_write<<<1, 1, 0, s>>>(flag + 0, trial + 1, 1000);  // more work after the record
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    // other stream, after the launch: wait on ev, then read the flag
    cudaStreamWaitEvent(s2, ev, 0);
    read_flag<<<1, 1, 0, s2>>>(flag, out);
    cudaDeviceSynchronize();
    if (*out != trial + 1) ++bad;
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  printf("wait-after-launch on an external record node: %d of 20 reads saw the old value\n", bad);
  return 0;
}
