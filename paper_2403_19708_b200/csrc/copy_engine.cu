// K1 / K4 — layer-wise pre-loader and asynchronous saver (copy engines over
// the host link), plus the ABI bookkeeping (version, last error).
//
// Each call turns one (session, layer) into a list of contiguous
// pinned-host <-> HBM segments and issues them as ONE cudaMemcpyBatchAsync on
// the caller's dedicated copy stream (one DMA descriptor list instead of one
// runtime call per block), then records the caller's event so the compute
// stream can wait on exactly that layer (overlap.py:69-123 / :126-200 model
// this schedule analytically; here it is real).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <string>
#include <vector>

#include "askv_internal.h"

namespace askv {

namespace {
thread_local std::string g_last_error;
}

void set_error(const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
}

void clear_error() { g_last_error.clear(); }

namespace {

// cudaMemcpyFlagPreferOverlapWithCompute is a tuning knob (ASKV_COPY_OVERLAP=1);
// default 0 keeps the DMAs on the copy engines.
unsigned copy_flags() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ASKV_COPY_OVERLAP");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v ? (unsigned)cudaMemcpyFlagPreferOverlapWithCompute : 0u;
}

// Issue a list of same-direction copies in stream order.
// Pointers are UVA-classified (cudaMemcpyDefault), so the same entry points
// serve a pinned-host arena (H2D / D2H over the host link) and an
// HBM-resident arena (D2D).
int issue_batch(std::vector<void*>& dsts, std::vector<void*>& srcs, std::vector<size_t>& sizes,
                cudaStream_t stream) {
  if (dsts.empty()) return ASKV_OK;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(stream, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone) {
    // inside a graph capture (the layer loop's HBM-tier copies): one memcpy
    // node per segment; the batch API is not capturable
    for (size_t i = 0; i < dsts.size(); ++i) {
      cudaError_t e = cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDefault, stream);
      if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync (captured)");
    }
    return ASKV_OK;
  }
  cudaMemcpyAttributes attr = {};
  attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
  attr.flags = copy_flags();
  size_t attr_idx = 0;
  size_t fail_idx = 0;
  cudaError_t e = cudaMemcpyBatchAsync(dsts.data(), srcs.data(), sizes.data(), dsts.size(),
                                       &attr, &attr_idx, 1, &fail_idx, stream);
  if (e == cudaSuccess) return ASKV_OK;
  // Batch API unavailable (older driver): same segments, one call each.
  (void)cudaGetLastError();
  for (size_t i = 0; i < dsts.size(); ++i) {
    e = cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDefault, stream);
    if (e != cudaSuccess) return cuda_status(e, "cudaMemcpyAsync");
  }
  return ASKV_OK;
}

// Small transfers done by SMs through UVA (pinned host memory is device
// addressable): token ids in, first token out.  They must not queue behind
// the multi-GB pre-load / save DMAs on the copy engines (which would put the
// whole pre-load of the next job in front of this job's 2 KB of token ids).
__global__ void copy_sm_kernel(uint8_t* __restrict__ dst, const uint8_t* __restrict__ src,
                               size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

}  // namespace
}  // namespace askv

using namespace askv;

extern "C" int askv_copy_sm(void* dst, const void* src, size_t bytes, void* stream) {
  clear_error();
  ASKV_REQUIRE(bytes <= (size_t)1 << 24, "copy_sm: %zu bytes is not a small transfer", bytes);
  if (bytes == 0) return ASKV_OK;
  ASKV_REQUIRE(dst && src, "copy_sm: null pointer");
  const int blocks = (int)((bytes + 255) / 256) < 64 ? (int)((bytes + 255) / 256) : 64;
  copy_sm_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(static_cast<uint8_t*>(dst),
                                                           static_cast<const uint8_t*>(src), bytes);
  return launch_status("copy_sm launch");
}

extern "C" int askv_version(void) { return 100; }

extern "C" const char* askv_last_error(void) { return g_last_error.c_str(); }

extern "C" int askv_preload_layer(void* dst, const void* host_base, const int64_t* block_ids,
                                  int nblocks, int64_t block_bytes, int64_t layer_off,
                                  int64_t chunk_bytes, int64_t tail_bytes, void* stream,
                                  void* done_event) {
  clear_error();
  ASKV_REQUIRE(nblocks >= 0 && chunk_bytes > 0 && block_bytes > 0 && layer_off >= 0,
               "preload: bad nblocks=%d chunk=%lld block=%lld layer_off=%lld", nblocks,
               (long long)chunk_bytes, (long long)block_bytes, (long long)layer_off);
  ASKV_REQUIRE(layer_off + chunk_bytes <= block_bytes, "preload: layer chunk outside block");
  ASKV_REQUIRE(tail_bytes >= 0 && tail_bytes <= chunk_bytes, "preload: bad tail_bytes");
  ASKV_REQUIRE(nblocks == 0 || (dst && host_base && block_ids), "preload: null pointer");
  std::vector<void*> d(nblocks), s(nblocks);
  std::vector<size_t> n(nblocks);
  auto* hb = static_cast<const char*>(host_base);
  auto* db = static_cast<char*>(dst);
  for (int i = 0; i < nblocks; ++i) {
    ASKV_REQUIRE(block_ids[i] >= 0, "preload: negative block id");
    d[i] = db + (int64_t)i * chunk_bytes;
    s[i] = const_cast<char*>(hb + block_ids[i] * block_bytes + layer_off);
    n[i] = (size_t)((i == nblocks - 1 && tail_bytes > 0) ? tail_bytes : chunk_bytes);
  }
  int rc = issue_batch(d, s, n, (cudaStream_t)stream);
  if (rc) return rc;
  if (done_event)
    return cuda_status(cudaEventRecord((cudaEvent_t)done_event, (cudaStream_t)stream),
                       "preload event record");
  return ASKV_OK;
}

extern "C" int askv_save_layer(void* host_base, const int64_t* block_ids, int nblocks,
                               int64_t block_bytes, int64_t layer_off, int block_tokens,
                               int64_t row_bytes, int64_t first_token, int n_tokens,
                               const void* src, void* stream, void* done_event) {
  clear_error();
  ASKV_REQUIRE(n_tokens >= 0 && block_tokens > 0 && row_bytes > 0 && first_token >= 0,
               "save: bad n_tokens=%d block_tokens=%d row_bytes=%lld first=%lld", n_tokens,
               block_tokens, (long long)row_bytes, (long long)first_token);
  ASKV_REQUIRE(layer_off + block_tokens * row_bytes <= block_bytes,
               "save: layer chunk outside block");
  const int64_t last = first_token + n_tokens;  // exclusive
  ASKV_REQUIRE(n_tokens == 0 || (last + block_tokens - 1) / block_tokens <= nblocks,
               "save: tokens [%lld,%lld) need more than %d blocks", (long long)first_token,
               (long long)last, nblocks);
  ASKV_REQUIRE(n_tokens == 0 || (host_base && block_ids && src), "save: null pointer");
  std::vector<void*> d, s;
  std::vector<size_t> n;
  auto* hb = static_cast<char*>(host_base);
  auto* sb = static_cast<const char*>(src);
  int64_t t = first_token;
  while (t < last) {
    const int64_t b = t / block_tokens;
    const int64_t r = t - b * block_tokens;
    int64_t cnt = block_tokens - r;
    if (cnt > last - t) cnt = last - t;
    ASKV_REQUIRE(block_ids[b] >= 0, "save: negative block id");
    d.push_back(hb + block_ids[b] * block_bytes + layer_off + r * row_bytes);
    s.push_back(const_cast<char*>(sb + (t - first_token) * row_bytes));
    n.push_back((size_t)(cnt * row_bytes));
    t += cnt;
  }
  int rc = issue_batch(d, s, n, (cudaStream_t)stream);
  if (rc) return rc;
  if (done_event)
    return cuda_status(cudaEventRecord((cudaEvent_t)done_event, (cudaStream_t)stream),
                       "save event record");
  return ASKV_OK;
}
