// In-kernel timeline of the K3 attention kernel: builds attention.cu with
// ASKV_ATTN_TRACE and prints, per CTA, globaltimer stamps (ns) relative to the
// earliest CTA start: entry, TMEM ready, Q landed (MMA warp), per-tile
// S-ready / P-done for softmax WG0, epilogue start, exit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DASKV_ATTN_TRACE \
//        -Ipaper_2403_19708_b200/csrc tools/attn_trace.cu -o tools/attn_trace -lcuda
#include "../paper_2403_19708_b200/csrc/attention.cu"

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

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
  const int kept = argc > 1 ? atoi(argv[1]) : 2869;
  const int n = argc > 2 ? atoi(argv[2]) : 301;
  const int hq = argc > 3 ? atoi(argv[3]) : 40;
  const int hkv = hq, d = 128;
  const int rows = kept + n;
  void *q, *kv, *out, *ws;
  cudaMalloc(&q, (size_t)n * hq * d * 2);
  cudaMalloc(&kv, (size_t)rows * 2 * hkv * d * 2);
  cudaMalloc(&out, (size_t)n * hq * d * 2);
  fill_bf16<<<1184, 256>>>((__nv_bfloat16*)q, (size_t)n * hq * d, 7u);
  fill_bf16<<<1184, 256>>>((__nv_bfloat16*)kv, (size_t)rows * 2 * hkv * d, 11u);
  const int splits = askv_attn_num_splits(kept, n, hq, 0);
  const size_t wsb = askv_attn_workspace_bytes(kept, n, hq, d, splits);
  cudaMalloc(&ws, wsb + 16);
  const int ctas = ((n + 127) / 128) * hq * splits;
  unsigned long long* tr;
  cudaMalloc(&tr, (size_t)ctas * 256 * 8);
  cudaMemcpyToSymbol(askv::g_attn_trace, &tr, sizeof(tr));
  for (int rep = 0; rep < 5; ++rep) {
    cudaMemset(tr, 0, (size_t)ctas * 256 * 8);
    int rc = askv_prefill_attn(q, kv, 2LL * hkv * d, kept, n, hq, hkv, d, 0.088f, out, ws, wsb,
                               splits, nullptr);
    if (rc) { printf("rc %d %s\n", rc, g_err); return 1; }
    cudaDeviceSynchronize();
  }
  std::vector<unsigned long long> h((size_t)ctas * 256);
  cudaMemcpy(h.data(), tr, h.size() * 8, cudaMemcpyDeviceToHost);
  unsigned long long t0 = ~0ull, tend = 0;
  int used = 0;  // CTAs that ran (the buffer is sized for one query tile per CTA)
  for (int c = 0; c < ctas; ++c) {
    if (!h[c * 256]) continue;
    used = c + 1;
    t0 = std::min(t0, h[c * 256]);
    tend = std::max(tend, h[c * 256 + 4]);
  }
  const int ran = used;
  printf("kept=%d n=%d hq=%d splits=%d ctas=%d span %.2f us\n", kept, n, hq, splits, ctas,
         (tend - t0) * 1e-3);
  double s_entry = 0, s_tmem = 0, s_q = 0, s_first = 0, s_loop = 0, s_epi = 0, s_exit = 0;
  int cnt = 0;
  for (int c = 0; c < ctas; ++c) {
    const unsigned long long* r = &h[c * 256];
    if (!r[3]) continue;
    ++cnt;
    s_entry += r[0] - t0;
    s_tmem += r[1] - r[0];
    s_q += r[2] - r[1];
    s_first += r[8] - r[1];
    int last = 0;
    for (int t = 0; t < 28; ++t) if (r[9 + 2 * t]) last = t;
    s_loop += r[9 + 2 * last] - r[8];
    s_epi += r[3] - r[9 + 2 * last];
    s_exit += r[4] - r[3];
  }
  printf("avg over %d CTAs (us): start offset %.2f | entry->tmem %.2f | tmem->Q %.2f | "
         "tmem->first S %.2f | WG0 tile loop %.2f | last tile->epilogue %.2f | epilogue->exit %.2f\n",
         cnt, s_entry / cnt * 1e-3, s_tmem / cnt * 1e-3, s_q / cnt * 1e-3, s_first / cnt * 1e-3,
         s_loop / cnt * 1e-3, s_epi / cnt * 1e-3, s_exit / cnt * 1e-3);
  for (int c : {0, 1, ran / 2, ran - 1}) {
    const unsigned long long* r = &h[c * 256];
    printf("cta %d: entry %.2f tmem %.2f q %.2f |", c, (r[0] - t0) * 1e-3, (r[1] - t0) * 1e-3,
           (r[2] - t0) * 1e-3);
    for (int t = 0; t < 28 && r[8 + 2 * t]; ++t)
      printf(" [%.2f %.2f]", (r[8 + 2 * t] - t0) * 1e-3, (r[9 + 2 * t] - t0) * 1e-3);
    printf(" | epi %.2f merged %.2f stored %.2f synced %.2f exit %.2f\n", (r[3] - t0) * 1e-3,
           r[5] ? (r[5] - t0) * 1e-3 : 0.0, r[6] ? (r[6] - t0) * 1e-3 : 0.0,
           r[7] ? (r[7] - t0) * 1e-3 : 0.0, (r[4] - t0) * 1e-3);
    printf("   WG0 P-done of warps 1..3 for tiles 0..3:");
    for (int t = 0; t < 4; ++t)
      printf(" [%.2f %.2f %.2f]", r[180 + 3 * t] ? (r[180 + 3 * t] - t0) * 1e-3 : 0.0,
             r[181 + 3 * t] ? (r[181 + 3 * t] - t0) * 1e-3 : 0.0,
             r[182 + 3 * t] ? (r[182 + 3 * t] - t0) * 1e-3 : 0.0);
    printf("\n");
    printf("   mma: P(j) seen / V(j) ready / PV(j) issued / K(j+2) ready:");
    for (int t = 0; t < 28 && r[64 + t]; ++t)
      printf(" [%.2f %.2f %.2f %.2f]", (r[64 + t] - t0) * 1e-3, (r[96 + t] - t0) * 1e-3,
             (r[160 + t] - t0) * 1e-3, r[128 + t] ? (r[128 + t] - t0) * 1e-3 : 0.0);
    printf("\n");
  }
  return 0;
}
