// In-kernel timeline of the stream-K attention kernel (attn_sk_kernel): builds
// attention.cu with ASKV_ATTN_TRACE and prints, for a few CTAs, globaltimer
// stamps (us from the earliest CTA entry): entry, TMEM ready, per piece the
// MMA warp's Q-ready / S-O-free, WG0's per-tile [S ready, P done], and the MMA
// warp's per-tile [P seen, V ready, PV issued, K(j+2) ready].
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE \
//        -Ipaper_2403_19708_b200/csrc tools/attn_sk_trace.cu -o /tmp/attn_sk_trace -lcuda
#include "../paper_2403_19708_b200/csrc/attention.cu"

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
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
  const int kept = argc > 1 ? atoi(argv[1]) : 2142;
  const int n = argc > 2 ? atoi(argv[2]) : 237;
  const int hq = argc > 3 ? atoi(argv[3]) : 40;
  const int hkv = hq, d = 128;
  const int rows = kept + n;
  void *q, *kv, *out, *ws;
  cudaMalloc(&q, (size_t)n * hq * d * 2);
  cudaMalloc(&kv, (size_t)rows * 2 * hkv * d * 2);
  cudaMalloc(&out, (size_t)n * hq * d * 2);
  fill_bf16<<<1184, 256>>>((__nv_bfloat16*)q, (size_t)n * hq * d, 7u);
  fill_bf16<<<1184, 256>>>((__nv_bfloat16*)kv, (size_t)rows * 2 * hkv * d, 11u);
  const size_t wsb = askv_attn_workspace_bytes_gqa(kept, n, hq, hkv, d, 0);
  cudaMalloc(&ws, wsb + 16);
  const int ctas = 160;
  unsigned long long* tr;
  cudaMalloc(&tr, (size_t)ctas * 256 * 8);
  cudaMemcpyToSymbol(askv::g_attn_trace, &tr, sizeof(tr));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(tr, 0, (size_t)ctas * 256 * 8);
    cudaEventRecord(e0);
    int rc = askv_prefill_attn(q, kv, 2LL * hkv * d, kept, n, hq, hkv, d, 0.088f, out, ws, wsb,
                               0, nullptr);
    cudaEventRecord(e1);
    if (rc) { printf("rc %d %s\n", rc, g_err); return 1; }
    cudaDeviceSynchronize();
    cudaEventElapsedTime(&ms, e0, e1);
  }
  std::vector<unsigned long long> h((size_t)ctas * 256);
  cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, tend = 0;
  int ran = 0;
  for (int c = 0; c < ctas; ++c) {
    if (!h[c * 256]) continue;
    ran = c + 1;
    t0 = std::min(t0, h[c * 256]);
    tend = std::max(tend, h[c * 256 + 4]);
  }
  printf("kept=%d n=%d hq=%d ctas=%d span %.2f us (events %.2f us incl. combine)\n", kept, n,
         hq, ran, (tend - t0) * 1e-3, ms * 1e3);
  auto us = [&](unsigned long long v) { return v ? (v - t0) * 1e-3 : -1.0; };
  std::vector<double> ent, tm, ex;
  for (int c = 0; c < ran; ++c) {
    const unsigned long long* r = &h[c * 256];
    ent.push_back(us(r[0]));
    tm.push_back(us(r[1]));
    ex.push_back(us(r[4]));
  }
  std::sort(ent.begin(), ent.end());
  std::sort(tm.begin(), tm.end());
  std::sort(ex.begin(), ex.end());
  printf("entry  min %.2f p50 %.2f max %.2f\n", ent[0], ent[ran / 2], ent[ran - 1]);
  printf("tmem   min %.2f p50 %.2f max %.2f\n", tm[0], tm[ran / 2], tm[ran - 1]);
  printf("exit   min %.2f p50 %.2f max %.2f\n", ex[0], ex[ran / 2], ex[ran - 1]);
  for (int c : {0, 1, ran / 2, ran - 1}) {
    const unsigned long long* r = &h[c * 256];
    printf("cta %d: entry %.2f tmem %.2f | pieces (q, o_free):", c, us(r[0]), us(r[1]));
    for (int k = 0; k < 4 && r[40 + 2 * k]; ++k) printf(" [%.2f %.2f]", us(r[40 + 2 * k]), us(r[41 + 2 * k]));
    printf(" | WG0 tiles:");
    for (int t = 0; t < 14 && r[8 + 2 * t]; ++t) printf(" [%.2f %.2f]", us(r[8 + 2 * t]), us(r[9 + 2 * t]));
    printf(" | last epi %.2f exit %.2f\n", us(r[3]), us(r[4]));
    printf("   last piece: merged %.2f partial stored %.2f fenced %.2f counted %.2f staged %.2f "
           "stored %.2f softmax-done %.2f\n", us(r[176]), us(r[177]), us(r[178]), us(r[179]),
           us(r[180]), us(r[181]), us(r[182]));
    printf("   mma [P seen, V ready, PV issued, K(j+2) ready]:");
    for (int t = 0; t < 28 && r[64 + t]; ++t)
      printf(" [%.2f %.2f %.2f %.2f]", us(r[64 + t]), us(r[96 + t]), us(r[160 + t]), us(r[128 + t]));
    printf("\n");
  }
  return 0;
}
