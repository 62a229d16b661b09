// K1 / K4 — layer-wise pre-loader and asynchronous saver (copy engines over
// the host link), plus the ABI bookkeeping (version, last error).
//
// Each call turns one (session, layer) into a list of contiguous
// pinned-host <-> HBM segments and issues them on the caller's dedicated copy
// stream: a run of consecutive arena blocks (same stride on both sides) is
// ONE strided cudaMemcpy2DAsync, an isolated segment one cudaMemcpyAsync, so a
// (session, layer) costs a handful of runtime calls, not one per block.  The
// caller's event is then recorded so the compute stream can wait on exactly
// that layer (overlap.py:69-123 / :126-200 model this schedule analytically;
// here it is real).
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

// ASKV_COPY_2D=0 disables the strided (2-D) form: every segment is its own
// cudaMemcpyAsync (an A/B knob for the DMA efficiency of short chunks).
bool use_2d() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("ASKV_COPY_2D");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

// One copy segment: `rows` equal pieces of `width` bytes, piece i at
// dst + i*dpitch / src + i*spitch (rows == 1: a plain contiguous copy).
struct Seg {
  char* dst;
  const char* src;
  size_t width, rows, dpitch, spitch;
};

// Append a contiguous piece, merging it into the previous segment when it
// continues it (contiguous on both sides, or one more row of the same stride).
void push_piece(std::vector<Seg>& v, char* d, const char* s, size_t n) {
  if (!v.empty()) {
    Seg& p = v.back();
    if (p.rows == 1 && p.dst + p.width == d && p.src + p.width == s) {
      p.width += n;  // contiguous continuation
      return;
    }
    if (use_2d() && n == p.width) {
      const char* plast_s = p.src + (p.rows - 1) * p.spitch;
      char* plast_d = p.dst + (p.rows - 1) * p.dpitch;
      if (p.rows == 1 && d > p.dst && s > p.src) {
        p.dpitch = (size_t)(d - p.dst);
        p.spitch = (size_t)(s - p.src);
        p.rows = 2;
        return;
      }
      if (p.rows > 1 && d == plast_d + p.dpitch && s == plast_s + p.spitch) {
        ++p.rows;
        return;
      }
    }
  }
  v.push_back(Seg{d, s, n, 1, n, n});
}

// Issue the segments in stream order.  Pointers are UVA-classified
// (cudaMemcpyDefault), so the same entry points serve a pinned-host arena
// (H2D / D2H over the host link) and an HBM-resident arena (D2D); inside a
// graph capture (the layer loop's HBM-tier copies) each becomes a memcpy node.
int issue(const std::vector<Seg>& v, cudaStream_t stream) {
  for (const Seg& g : v) {
    cudaError_t e;
    if (g.rows == 1)
      e = cudaMemcpyAsync(g.dst, g.src, g.width, cudaMemcpyDefault, stream);
    else
      e = cudaMemcpy2DAsync(g.dst, g.dpitch, g.src, g.spitch, g.width, g.rows,
                            cudaMemcpyDefault, stream);
    if (e != cudaSuccess) return cuda_status(e, g.rows == 1 ? "cudaMemcpyAsync" : "cudaMemcpy2DAsync");
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
  std::vector<Seg> segs;
  segs.reserve(4);
  auto* hb = static_cast<const char*>(host_base);
  auto* db = static_cast<char*>(dst);
  for (int i = 0; i < nblocks; ++i) {
    ASKV_REQUIRE(block_ids[i] >= 0, "preload: negative block id");
    push_piece(segs, db + (int64_t)i * chunk_bytes, hb + block_ids[i] * block_bytes + layer_off,
               (size_t)((i == nblocks - 1 && tail_bytes > 0) ? tail_bytes : chunk_bytes));
  }
  int rc = issue(segs, (cudaStream_t)stream);
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
  std::vector<Seg> segs;
  auto* hb = static_cast<char*>(host_base);
  auto* sb = static_cast<const char*>(src);
  int64_t t = first_token;
  while (t < last) {
    const int64_t b = t / block_tokens;
    const int64_t r = t - b * block_tokens;
    int64_t cnt = block_tokens - r;
    if (cnt > last - t) cnt = last - t;
    ASKV_REQUIRE(block_ids[b] >= 0, "save: negative block id");
    push_piece(segs, hb + block_ids[b] * block_bytes + layer_off + r * row_bytes,
               sb + (t - first_token) * row_bytes, (size_t)(cnt * row_bytes));
    t += cnt;
  }
  int rc = issue(segs, (cudaStream_t)stream);
  if (rc) return rc;
  if (done_event)
    return cuda_status(cudaEventRecord((cudaEvent_t)done_event, (cudaStream_t)stream),
                       "save event record");
  return ASKV_OK;
}

// K4 for a whole job: every layer's save in one call (the saver IO thread
// otherwise pays ~5 runtime calls through ctypes per layer, which at 16 jobs x
// 40 layers per batched pass made the host the bottleneck).  Layers are saved
// in groups of up to G (ASKV_SAVE_GROUP, default 8) whose write-buffer slots
// sit at a constant stride: one 2-D DMA per block piece covers the group's
// layers (host pitch = the block's layer chunk), so a 301-token turn moves
// ~16 MB pieces instead of ~2 MB ones -- the link gives small D2H pieces far
// less while the pre-loader's H2D runs (profiles/r02_link_probe.txt).  Per
// group: wait ev_ready of its layers (the loop's rope_new wrote the rows),
// the DMAs bracketed by its first layer's timing events ev_t0 / ev_t1 (the
// other layers get zero-length intervals at the group's end), ev_done of
// every layer in it (the slots are free again); then ev_last.
static int save_group_knob() {
  static int g = -1;
  if (g < 0) {
    const char* e = getenv("ASKV_SAVE_GROUP");
    g = e ? atoi(e) : 8;
    if (g < 1) g = 1;
  }
  return g;
}

extern "C" int askv_save_layers(void* host_base, const int64_t* block_ids, int nblocks,
                                int64_t block_bytes, int64_t chunk_bytes, int layers,
                                int block_tokens, int64_t row_bytes, int64_t first_token,
                                int n_tokens, const void* const* src, void* const* ev_ready,
                                void* const* ev_done, void* const* ev_t0, void* const* ev_t1,
                                void* ev_last, void* stream) {
  clear_error();
  ASKV_REQUIRE(layers > 0 && src != nullptr, "save_layers: bad layers=%d", layers);
  cudaStream_t s = (cudaStream_t)stream;
  const int gmax = save_group_knob();
  auto rec = [&](void* const* evs, int l) {
    if (evs && evs[l]) cudaEventRecord((cudaEvent_t)evs[l], s);
  };
  for (int l0 = 0; l0 < layers;) {
    // the group: consecutive layers whose sources are a constant stride apart
    int l1 = l0 + 1;
    const int64_t stride = l0 + 1 < layers ? static_cast<const char*>(src[l0 + 1]) -
                                                 static_cast<const char*>(src[l0])
                                           : 0;
    while (l1 < layers && l1 - l0 < gmax && stride > 0 &&
           static_cast<const char*>(src[l1]) - static_cast<const char*>(src[l1 - 1]) == stride)
      ++l1;
    for (int l = l0; l < l1; ++l) {
      if (ev_ready && ev_ready[l]) {
        const int rc = cuda_status(cudaStreamWaitEvent(s, (cudaEvent_t)ev_ready[l], 0),
                                   "save_layers wait");
        if (rc) return rc;
      }
    }
    rec(ev_t0, l0);
    if (l1 - l0 == 1) {
      const int rc = askv_save_layer(host_base, block_ids, nblocks, block_bytes,
                                     (int64_t)l0 * chunk_bytes, block_tokens, row_bytes,
                                     first_token, n_tokens, src[l0], stream, nullptr);
      if (rc) return rc;
    } else {
      ASKV_REQUIRE(n_tokens >= 0 && block_tokens > 0 && row_bytes > 0 && first_token >= 0,
                   "save_layers: bad n_tokens=%d", n_tokens);
      ASKV_REQUIRE((int64_t)(l1 - 1) * chunk_bytes + block_tokens * row_bytes <= block_bytes,
                   "save_layers: layer chunk outside block");
      const int64_t last = first_token + n_tokens;
      ASKV_REQUIRE(n_tokens == 0 || (last + block_tokens - 1) / block_tokens <= nblocks,
                   "save_layers: tokens need more than %d blocks", nblocks);
      ASKV_REQUIRE(n_tokens == 0 || (host_base && block_ids), "save_layers: null pointer");
      auto* hb = static_cast<char*>(host_base) + (int64_t)l0 * chunk_bytes;
      auto* sb = static_cast<const char*>(src[l0]);
      for (int64_t t = first_token; t < last;) {
        const int64_t b = t / block_tokens;
        const int64_t r = t - b * block_tokens;
        int64_t cnt = block_tokens - r;
        if (cnt > last - t) cnt = last - t;
        ASKV_REQUIRE(block_ids[b] >= 0, "save_layers: negative block id");
        const cudaError_t e = cudaMemcpy2DAsync(
            hb + block_ids[b] * block_bytes + r * row_bytes, (size_t)chunk_bytes,
            sb + (t - first_token) * row_bytes, (size_t)stride, (size_t)(cnt * row_bytes),
            (size_t)(l1 - l0), cudaMemcpyDefault, s);
        if (e != cudaSuccess) return cuda_status(e, "save_layers cudaMemcpy2DAsync");
        t += cnt;
      }
    }
    for (int l = l0; l < l1; ++l) rec(ev_done, l);
    rec(ev_t1, l0);
    for (int l = l0 + 1; l < l1; ++l) {  // zero-length intervals: the group's time is l0's
      rec(ev_t0, l);
      rec(ev_t1, l);
    }
    l0 = l1;
  }
  if (ev_last)
    return cuda_status(cudaEventRecord((cudaEvent_t)ev_last, s), "save_layers event record");
  return ASKV_OK;
}
