// Build-time A/B timing of K3: compile attention.cu with -D knobs, time
// askv_prefill_attn at the path's shapes (median of 50 launches, CUDA events,
// 256 MB L2 flush before each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 [-DKNOB=..] \
//        -Ipaper_2403_19708_b200/csrc -Iinclude tools/attn_ab.cu -o /tmp/attn_ab -lcuda
#include "../paper_2403_19708_b200/csrc/attention.cu"

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <vector>

static char g_err[512];
namespace askv {
void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void clear_error() { g_err[0] = 0; }
}  // namespace askv

__global__ void fill_bf16(__nv_bfloat16* p, size_t n, uint32_t seed) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    x ^= x >> 13;
    x *= 0x5bd1e995u;
    x ^= x >> 15;
    p[i] = __float2bfloat16(((int)(x & 0xffff) - 32768) * (2.0f / 32768.f));
  }
}

int main(int argc, char** argv) {
  const char* tag = argc > 1 ? argv[1] : "";
  const int shapes[][4] = {{2142, 237, 40, 40}, {2869, 301, 40, 40}, {1000, 100, 40, 40},
                           {3600, 700, 40, 40}, {2048, 256, 8, 1}};
  void* flush;
  cudaMalloc(&flush, 256 << 20);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (auto& sh : shapes) {
    const int kept = sh[0], n = sh[1], hq = sh[2], hkv = sh[3], d = 128;
    void *q, *kv, *out, *ws;
    cudaMalloc(&q, (size_t)n * hq * d * 2);
    cudaMalloc(&kv, (size_t)(kept + n) * 2 * hkv * d * 2);
    cudaMalloc(&out, (size_t)n * hq * d * 2);
    fill_bf16<<<1184, 256>>>((__nv_bfloat16*)q, (size_t)n * hq * d, 7u);
    fill_bf16<<<1184, 256>>>((__nv_bfloat16*)kv, (size_t)(kept + n) * 2 * hkv * d, 11u);
    const int splits = askv_attn_num_splits_gqa(kept, n, hq, hkv, 0);
    const size_t wsb = askv_attn_workspace_bytes_gqa(kept, n, hq, hkv, d, splits);
    cudaMalloc(&ws, wsb + 16);
    std::vector<float> ts;
    for (int rep = 0; rep < 55; ++rep) {
      cudaMemsetAsync(flush, rep, 256 << 20);
      cudaEventRecord(e0);
      int rc = askv_prefill_attn(q, kv, 2LL * hkv * d, kept, n, hq, hkv, d, 0.088f, out, ws, wsb,
                                 splits, nullptr);
      cudaEventRecord(e1);
      if (rc) { printf("rc %d %s\n", rc, g_err); return 1; }
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep >= 5) ts.push_back(ms * 1e3f);
    }
    std::sort(ts.begin(), ts.end());
    const double fl = 4.0 * hq * d * ((double)n * kept + (double)n * (n + 1) / 2);
    printf("%s kept=%d n=%d hq=%d hkv=%d splits=%d  %.2f us  %.0f TF/s\n", tag, kept, n, hq, hkv,
           splits, ts[ts.size() / 2], fl / (ts[ts.size() / 2] * 1e-6) / 1e12);
    cudaFree(q); cudaFree(kv); cudaFree(out); cudaFree(ws);
  }
  return 0;
}
