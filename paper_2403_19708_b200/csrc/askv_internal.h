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
// K5: in-place / out-of-place bf16 sum over a NCCL communicator (collective.cu).
int tp_allreduce_bf16(const void* send, void* recv, int64_t elems, void* comm,
                      cudaStream_t stream);
// K3's optional V source: the V rows of the first `tiles` 128-row KV tiles
// are read where the pre-loader left them instead of from `kv` (K2 then
// copies no V for those rows).  kind 1: contiguous rows (a read-buffer slot),
// tile t at row row0 + 128 t of `base`; kind 2: HBM-arena block table, tile t
// = block t at row blk_off[t] / row_elems + layer_row of `base` (`rows` rows).
struct VSource {
  int kind = 0;
  int tiles = 0;
  const void* base = nullptr;
  int64_t rows = 0;
  int64_t row0 = 0;
  const int64_t* blk_off = nullptr;
  int64_t row_elems = 0;
  int64_t layer_row = 0;
};
// K3 over a batch of jobs in one launch (askv_prefill_layers_batch): job i's
// queries are rows [q_row0, q_row0 + n_new) of q, its keys / values rows
// [kv_row0, kv_row0 + n_cached + n_new) of kv; optional V source shared by
// the jobs (an HBM arena: kind 2, per-job block tables).
struct VarlenBatch {
  int n = 0;
  const void* q = nullptr;
  const void* kv = nullptr;
  int64_t kv_row_stride = 0;
  int hq = 0, hkv = 0, head_dim = 0;
  float scale = 1.f;
  const int* n_new = nullptr;
  const int* n_cached = nullptr;
  const int* q_row0 = nullptr;
  const int* kv_row0 = nullptr;
  void* const* out = nullptr;
  const void* vsrc_base = nullptr;
  int64_t vsrc_rows = 0, vsrc_row_elems = 0, v_layer_row = 0;
  const int* v_src_tiles = nullptr;
  const int64_t* const* v_blk_off = nullptr;
};
int prefill_attn_varlen(const VarlenBatch& b, void* stream, unsigned long long* stamp);
int prefill_attn_stamped(const void* q, const void* kv, int64_t kv_row_stride, int n_cached,
                         int n_new, int n_heads, int n_kv_heads, int head_dim, float scale,
                         void* out, void* workspace, size_t workspace_bytes, int num_splits,
                         void* stream, unsigned long long* stamp,
                         const VSource* vsrc = nullptr);
int rmsnorm_stamped(const void* x, const void* w, void* y, int rows, int cols, float eps,
                    void* stream, unsigned long long* begin);
int rope_new_stamped(const void* qkv, int64_t qkv_row_stride, int n_new, int n_heads,
                     int n_kv_heads, int head_dim, const float* rope_table, int table_positions,
                     int pos0, void* q_out, void* kv_out, int64_t kv_row_stride, void* save_out,
                     void* stream, unsigned long long* end);
// rope_new for a batch of jobs in one launch (their new tokens consecutive
// in qkv / q_out; per job its first position and K|V / save destinations).
int rope_new_batch(const void* qkv, int64_t qkv_row_stride, int n_jobs, const int* n_new,
                   const int* pos0, int n_heads, int n_kv_heads, int head_dim,
                   const float* rope_table, int table_positions, void* q_out,
                   void* const* kv_out, int64_t kv_row_stride, void* const* save_out,
                   void* stream, unsigned long long* end);
int reembed_stamped(const void* src_base, const int64_t* src_block_off, int block_tokens,
                    int64_t src_row_stride, int64_t first_token, int kept, int n_kv_heads,
                    int head_dim, const float* rope_table, int table_positions,
                    const int32_t* positions, int pos0, void* dst, int64_t dst_row_stride,
                    void* stream, unsigned long long* stamp, int v_from = 0);
// K2 for a batch of HBM-arena sessions in one launch (shared source arena
// layer base, strides and RoPE table; per job its block table, first stored
// token, kept rows, first position, V-copy start and destination rows).
int reembed_batch(const void* src_base, int block_tokens, int64_t src_row_stride, int n_jobs,
                  const int64_t* const* blk_off, const int64_t* first_token, const int* kept,
                  const int* pos0, const int* v_from, void* const* dst, int64_t dst_row_stride,
                  int n_kv_heads, int head_dim, const float* rope_table, int table_positions,
                  void* stream, unsigned long long* stamp);

}  // namespace askv
