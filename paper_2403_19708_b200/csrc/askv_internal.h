// Internal helpers shared by the C-ABI translation units.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include <cstdarg>
#include <cstdio>
#include <string>

#include "../../include/askv.h"

namespace askv {

void set_error(const char* fmt, ...);
void clear_error();

inline int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return ASKV_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return ASKV_ECUDA;
}

inline int launch_status(const char* what) { return cuda_status(cudaGetLastError(), what); }

#define ASKV_REQUIRE(cond, ...)          \
  do {                                   \
    if (!(cond)) {                       \
      ::askv::set_error(__VA_ARGS__);    \
      return ASKV_EINVAL;                \
    }                                    \
  } while (0)

// Entry points of the native layer loop with in-kernel launch timestamps
// ({begin, end} globaltimer ns, see attention.cu launch_stamp_*); the C ABI
// functions call these with stamp == nullptr.
int prefill_attn_stamped(const void* q, const void* kv, int64_t kv_row_stride, int n_cached,
                         int n_new, int n_heads, int n_kv_heads, int head_dim, float scale,
                         void* out, void* workspace, size_t workspace_bytes, int num_splits,
                         void* stream, unsigned long long* stamp);
int rmsnorm_stamped(const void* x, const void* w, void* y, int rows, int cols, float eps,
                    void* stream, unsigned long long* begin);
int rope_new_stamped(const void* qkv, int64_t qkv_row_stride, int n_new, int n_heads,
                     int n_kv_heads, int head_dim, const float* rope_table, int table_positions,
                     int pos0, void* q_out, void* kv_out, int64_t kv_row_stride, void* save_out,
                     void* stream, unsigned long long* end);
int reembed_stamped(const void* src_base, const int64_t* src_block_off, int block_tokens,
                    int64_t src_row_stride, int64_t first_token, int kept, int n_kv_heads,
                    int head_dim, const float* rope_table, int table_positions,
                    const int32_t* positions, int pos0, void* dst, int64_t dst_row_stride,
                    void* stream, unsigned long long* stamp);

}  // namespace askv
