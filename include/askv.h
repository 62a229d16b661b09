/*
 * askv.h — C ABI of the B200 (sm_100a) AttentionStore KV-reuse prefill path.
 *
 * The reference (kvsim 0.1.0, /root/reference/pkg/src/kvsim) is pure Python
 * with no FFI; each entry point below names the reference interface whose
 * behaviour it implements for the hot path.  The Python host
 * package paper_2403_19708_b200 binds these with ctypes.
 *
 * Conventions
 *   - plain pointers and sizes; bf16 tensors are passed as void* (2-byte
 *     elements), device or pinned-host as documented per argument;
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy stream);
 *   - no allocation and no device synchronisation inside any call;
 *   - return 0 on success, ASKV_EINVAL for argument errors (ValueError in the
 *     Python shim), ASKV_ECUDA for CUDA launch/runtime errors (RuntimeError),
 *     ASKV_EUNSUPPORTED for shapes the kernels are not built for;
 *     askv_last_error() returns the message of the calling thread's last error;
 *   - deterministic: no atomics in reductions, fixed split-KV combine order.
 *
 * KV row layout (device and host): one token = [2][Hkv][head_dim] bf16,
 * K then V, "pre-RoPE" (keys stored before positional encoding).
 * Host arena: block b of a session holds `block_tokens` rows per layer;
 * the (block, layer) chunk is contiguous at host_base + block_id*block_bytes
 * + layer*chunk_bytes, chunk_bytes = block_tokens * row_bytes.
 */
#ifndef ASKV_H_
#define ASKV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASKV_OK 0
#define ASKV_EINVAL (-1)
#define ASKV_ECUDA (-2)
#define ASKV_EUNSUPPORTED (-3)

/* ABI version (major*100 + minor). */
int askv_version(void);

/* Message for the last non-zero return on this thread ("" if none). */
const char* askv_last_error(void);

/*
 * RoPE cos/sin table, computed in float64 and stored as float32 pairs:
 * table[p*(head_dim/2) + i] = (cos(p*theta^(-2i/d)), sin(...)), p in [0, max_pos).
 * Replaces: rope.py:55-60 (_pair_angles) + the cos/sin of rope.py:67-68.
 * table: device float[2*max_pos*(head_dim/2)].
 */
int askv_rope_table(float* table, int max_pos, int head_dim, double theta_base, void* stream);

/*
 * K2 — fused gather + truncate + re-embed of one layer of a session's cached
 * pre-RoPE K/V.  Row i (0 <= i < kept) is session token (first_token + i);
 * its source row lives in block (first_token+i)/block_tokens of `src_block_off`
 * (element offsets from src_base, device int64 array), or, when src_block_off
 * is NULL, at src_base + (first_token+i)*src_row_stride.  K is rotated at
 * position positions[i] (device int32; NULL = the compacted positions pos0 + i
 * used after truncation, rope.py:263-266) and written with V to
 * dst + i*dst_row_stride.  Truncation = the caller starts at first_token
 * (multiple of block_tokens after whole-block drops) and passes `kept`.
 * Replaces: rope.py:63-74 (rotate_matrix) at rope.py:138, KvRecord.truncated
 * rope.py:48-52, and the kept range of sim.py:468-483.
 * src/dst: device bf16.  Strides in elements.
 * Precondition: every positions[i] lies in [0, table_positions) -- the kernel
 * does not bound-check explicit positions (the pos0 form is checked; the
 * Python numeric API checks explicit ones, ops._check_positions).
 */
int askv_reembed(const void* src_base, const int64_t* src_block_off, int block_tokens,
                 int64_t src_row_stride, int64_t first_token, int kept, int n_kv_heads,
                 int head_dim, const float* rope_table, int table_positions,
                 const int32_t* positions, int pos0, void* dst, int64_t dst_row_stride,
                 void* stream);

/*
 * Rotate every head of n_rows rows x[i] = [heads][hd] at positions[i]
 * (device int32, or pos0 + i when NULL) into out[i].
 * Replaces: rope.py:63-74 (rotate_matrix) / rope.py:77-85 (rope_rotate).
 * Precondition as askv_reembed: explicit positions within [0, table_positions).
 */
int askv_rotate_rows(const void* x, int64_t x_row_stride, int n_rows, int n_heads,
                     int head_dim, const float* rope_table, int table_positions,
                     const int32_t* positions, int pos0, void* out, int64_t out_row_stride,
                     void* stream);

/*
 * New-token epilogue of the QKV projection: for token i < n_new of
 * qkv[i] = [q (Hq*hd) | k (Hkv*hd) | v (Hkv*hd)] (row stride qkv_row_stride):
 *   q_out[i]  = rope(q, pos0+i)            layout [n_new][Hq][hd]
 *   kv_out[i] = [rope(k, pos0+i) | v]      row i of a [rows][2][Hkv][hd] buffer
 *   save_out[i] = [k | v] pre-RoPE         (may be NULL)
 * Replaces: rope.py:139-140 (rotation of new k and q) and the paper's
 * "cache k, v before apply_pos_emb" order.
 */
int askv_rope_new(const void* qkv, int64_t qkv_row_stride, int n_new, int n_heads,
                  int n_kv_heads, int head_dim, const float* rope_table, int table_positions,
                  int pos0, void* q_out, void* kv_out, int64_t kv_row_stride, void* save_out,
                  void* stream);

/*
 * K3 — prefill attention over [reused prefix | new tokens] on tcgen05/TMEM,
 * TMA-fed.  num_splits <= 1 with single-tile units: stream-K (the KV tiles of
 * all (query tile, head) units cut into one equal range per SM, partials of
 * the units cut across SMs merged by a deterministic combine); num_splits > 1:
 * uniform split-KV + combine.
 *   q   : [n_new][Hq][hd] bf16 (already rotated)
 *   kv  : [n_cached+n_new][2][Hkv][hd] bf16 rows (K rotated), row stride kv_row_stride
 *   out : [n_new][Hq][hd] bf16
 * Query i sees keys j <= n_cached + i; q-head h uses kv-head h/(Hq/Hkv).
 * scale = 1/sqrt(hd) reproduces rope.py:98.  num_splits = 0 picks the schedule
 * for the SM count; workspace must hold askv_attn_workspace_bytes_gqa(...).
 * Replaces: rope.py:94-105 (_causal_attention) inside rope.py:118-144.
 */
int askv_prefill_attn(const void* q, const void* kv, int64_t kv_row_stride, int n_cached,
                      int n_new, int n_heads, int n_kv_heads, int head_dim, float scale,
                      void* out, void* workspace, size_t workspace_bytes, int num_splits,
                      void* stream);
size_t askv_attn_workspace_bytes_gqa(int n_cached, int n_new, int n_heads, int n_kv_heads,
                                     int head_dim, int num_splits);
/* The same without n_kv_heads: the largest need over every grouping of n_heads. */
size_t askv_attn_workspace_bytes(int n_cached, int n_new, int n_heads, int head_dim,
                                 int num_splits);
/* Split count the auto policy would use (for reporting / tests). */
int askv_attn_num_splits(int n_cached, int n_new, int n_heads, int sm_count);
/* Same with GQA: n_heads q-heads over n_kv_heads kv heads (the launch packs a
 * kv head's (token, q-head) rows into shared tiles). */
int askv_attn_num_splits_gqa(int n_cached, int n_new, int n_heads, int n_kv_heads, int sms);

/*
 * K1 — layer-wise pre-loader: H2D of one layer's kept blocks of one session
 * from the pinned host arena into a contiguous HBM read-buffer slot:
 *   dst + i*chunk_bytes <- host_base + block_ids[i]*block_bytes + layer_off
 * for i < nblocks (the last copy carries tail_bytes, 0 = full chunk), issued
 * as one batch on `stream`; records `done_event` (cudaEvent_t, may be NULL).
 * block_ids is a host array.
 * Replaces: the load stream of overlap.py:69-123 (plan_preload) as called from
 * sim.py:436-442.
 */
int askv_preload_layer(void* dst, const void* host_base, const int64_t* block_ids,
                       int nblocks, int64_t block_bytes, int64_t layer_off,
                       int64_t chunk_bytes, int64_t tail_bytes, void* stream,
                       void* done_event);

/*
 * K4 — layer-wise asynchronous saver: D2H of n_tokens new rows (contiguous
 * [n][row_bytes] at src, device) into the session's host blocks, starting at
 * session token `first_token` (block block_ids[t/block_tokens], row
 * t%block_tokens, layer offset layer_off).  One batch on `stream`; records
 * `done_event` if non-NULL.  block_ids is a host array covering the tail.
 * Replaces: overlap.py:126-200 (plan_async_save) and the save of sim.py:532-555.
 */
int askv_save_layer(void* host_base, const int64_t* block_ids, int nblocks,
                    int64_t block_bytes, int64_t layer_off, int block_tokens,
                    int64_t row_bytes, int64_t first_token, int n_tokens, const void* src,
                    void* stream, void* done_event);
/* K4 for all `layers` layers of a job in one call: src[l] holds layer l's
 * n_tokens rows.  Layers whose src are a constant stride apart are saved in
 * groups (ASKV_SAVE_GROUP, default 8) as one 2-D DMA per block piece: a
 * group waits every ev_ready[l] of its layers (may be NULL), brackets its
 * DMAs with its first layer's ev_t0 / ev_t1 (timing, may be NULL; the other
 * layers' pairs are recorded together after it, zero-length) and records
 * each layer's ev_done after them; ev_last after the last group.  Replaces:
 * the per-layer save slots of overlap.py:126-200 (one call instead of one
 * per layer). */
int askv_save_layers(void* host_base, const int64_t* block_ids, int nblocks, int64_t block_bytes,
                     int64_t chunk_bytes, int layers, int block_tokens, int64_t row_bytes,
                     int64_t first_token, int n_tokens, const void* const* src,
                     void* const* ev_ready, void* const* ev_done, void* const* ev_t0,
                     void* const* ev_t1, void* ev_last, void* stream);

/*
 * Small copy executed by SMs through unified addressing (pinned host <-> device):
 * keeps the few-KB per-job transfers (token ids in, first token out) off the
 * copy engines that are busy with the pre-loader / saver DMAs.  bytes <= 16 MiB.
 */
int askv_copy_sm(void* dst, const void* src, size_t bytes, void* stream);

/*
 * Fused elementwise ops of the LLaMA block the runner executes around the path
 * (no reference counterpart; the reference has no model):
 *   askv_rmsnorm : y[r] = x[r] * rsqrt(mean(x[r]^2) + eps) * w   (bf16 io, fp32 math)
 *   askv_silu_mul: out[r] = silu(gu[r][0:ffn]) * gu[r][ffn:2ffn]
 */
int askv_rmsnorm(const void* x, const void* w, void* y, int rows, int cols, float eps,
                 void* stream);
int askv_silu_mul(const void* gu, void* out, int rows, int ffn, void* stream);

/*
 * Native events (cudaEvent_t as void*) used by the runtime's streams / IO threads.
 */
int askv_event_create(void** ev, int timing);
int askv_event_destroy(void* ev);
int askv_event_record(void* ev, void* stream);
int askv_stream_wait_event(void* stream, void* ev);
int askv_event_elapsed_ms(void* start, void* end, float* ms);
/* Block the calling host thread until the event's recorded work is done (the
 * disk tier fences arena blocks on a session's in-flight copies with it). */
int askv_event_synchronize(void* ev);

/*
 * One job's full layer loop (the reuse prefill of N new tokens over `kept`
 * reused rows), issued natively: per layer rmsnorm, QKV GEMM (cuBLASLt),
 * rope_new (+ the pre-RoPE rows for the saver), wait for the pre-load event,
 * K2 re-embed (+ optional promotion into the HBM tier), K3 attention, O GEMM
 * with residual, rmsnorm, gate/up GEMM, silu*mul, down GEMM with residual.
 * Event arrays (length `layers`, entries may be NULL) connect it to the
 * pre-loader / saver streams.  With `allreduce` set (tensor parallelism) the
 * W_o / W_down partials go through the callback before the residual add.
 * Replaces: the per-layer composition the reference models as compute slots of
 * overlap.py:69-123 (one slot per layer, loads may lag one layer).
 */
typedef struct askv_prefill_plan {
  int32_t layers, d_model, n_heads, n_kv_heads, head_dim, ffn;
  int32_t n_new, kept, head;
  float rms_eps, attn_scale;
  int32_t attn_splits;
  const void* const* w_in;
  const void* const* w_qkv;
  const void* const* w_o;
  const void* const* w_post;
  const void* const* w_gu;
  const void* const* w_down;
  void* x;
  void* h;
  void* qkv;
  void* q_rot;
  void* kv;
  void* attn_out;
  void* gu;
  void* act;
  void* attn_ws;
  size_t attn_ws_bytes;
  void* gemm_ws;
  size_t gemm_ws_bytes;
  const float* rope_table;
  int32_t rope_positions;
  int32_t src_kind; /* 0 none, 1 contiguous per-layer rows, 2 block table */
  const void* const* src_layer;
  const int64_t* src_block_off;
  int32_t block_tokens;
  int64_t src_row_stride;
  void* const* ev_src_ready;
  void* const* ev_src_free;
  void* const* save_rows;
  void* const* ev_save_free;
  void* const* ev_save_ready;
  void* promote_base;
  const int64_t* promote_block_ids; /* host array */
  int32_t promote_nblocks;
  int64_t block_bytes, chunk_bytes, row_bytes;
  /* Optional device timestamps (globaltimer ns).  CUDA timing events cost
   * ~24 us each on a stream while the host link is saturated
   * (profiles/r01d_summary.md), so the kernels that bound each interval write
   * them themselves (start of CTA 0 / atomicMax of CTA ends); one 1-thread
   * stamp kernel marks the last layer's end.  Layout:
   *   stamps[0]                 loop begin (start of layer 0's input rmsnorm)   (flags & 1)
   *   stamps[1 + 7*l + 0]       layer l end (start of layer l+1's input rmsnorm) (flags & 1)
   *   stamps[1 + 7*l + 1]       pre-load wait begin (end of rope_new)  (flags & 1, ev_src_ready)
   *   stamps[1 + 7*l + 3 / 4]   K2 re-embed begin / end; the begin is also the
   *                             pre-load wait end  (flags & 2, or flags & 1 with ev_src_ready)
   *   stamps[1 + 7*l + 5 / 6]   K3 attention begin / end incl. the split-KV combine (flags & 2)
   * stamps[1 + 7*l + 2] is unused.  Entries whose stage does not run are left
   * untouched. */
  uint64_t* stamps;
  int32_t stamp_flags;
  void (*allreduce)(void* ptr, int64_t elems, void* stream, void* ctx);
  void* allreduce_ctx;
  /* Optional per-layer resident KV (rotated rows [0, kept + n_new) per layer,
   * row stride 2*Hkv*hd): when set, K2 / rope_new / K3 use kv_layers[l] instead
   * of the shared `kv` buffer, so the whole context stays resident for decode;
   * with src_kind 0 and kept > 0 the first `kept` rows are already there. */
  void* const* kv_layers;
  /* 1: capture the loop into a CUDA graph (cached per shape, updated in
   * place) and launch that; 0: issue every kernel on `stream`.  Ignored
   * (stream issue) with `allreduce` set. */
  int32_t graph;
  /* Optional second attention KV buffer (same size as `kv`).  When set, with a
   * pre-load source (src_kind 1/2), kv_layers NULL and neither allreduce nor
   * promote_base, layers alternate between kv and kv_alt and K2 of layer l+1
   * runs on a second stream alongside K3 of layer l, on the SMs K3 leaves idle
   * (the pre-load wait of layer l is then observed before K3, stamps[1+7l+5]
   * marks its end). */
  void* kv_alt;
  /* Optional HBM-tier write-through: right after rope_new,
   * copy the layer's new pre-RoPE rows (save_rows) into rows
   * [head + kept, head + kept + n_new) of these HBM-arena blocks, on `stream`,
   * so every access to the tier (this copy, promote_base, K2 reads) is in one
   * stream order. */
  void* mirror_base;
  const int64_t* mirror_block_ids; /* host array */
  int32_t mirror_nblocks;
  /* Optional NCCL communicator of the tensor-parallel group (config C5,
   * askv_nccl_comm_init).  When set, the row-parallel W_o and W_down partials
   * are summed by ncclAllReduce on `stream` inside the loop (captured into
   * the layer graph): rank `tp_rank` 0 adds the residual in its GEMM epilogue
   * and reduces in place in x; the other ranks reduce their partial from h
   * into x, so x = x + sum over ranks with no separate residual kernel. */
  void* nccl_comm;
  int32_t tp_rank;
  /* Rows addressable from the pre-load source for K3's direct V reads (0 =
   * off): src_kind 1 -- rows of each src_layer[l] slot; src_kind 2 -- rows of
   * the HBM arena from src_layer[0] on.  With it, the V rows of the kept
   * rows' whole 128-row tiles are read by K3 where the pre-loader left them
   * (src_kind 2 needs head 0 and block_tokens 128) and K2 moves K only: K2's
   * traffic is the rotation's own read + write of K. */
  int64_t src_rows;
} askv_prefill_plan;

int askv_prefill_layers(const askv_prefill_plan* plan, void* stream);
/* Several jobs (sessions' turns) in one pass over the layers: the norms,
 * projections and MLP run once over the jobs' concatenated new tokens, while
 * rope_new, the pre-load wait, K2 and K3 run per job on its own rows.  plans[i]
 * describes job i as for askv_prefill_layers; the jobs share the model and
 * their x / h / qkv / q_rot / attn_out / gu / act buffers are consecutive
 * slices of plans[0]'s (job i's starts after jobs 0..i-1's rows); job 0's
 * stamps carry the layer timeline.  No tensor parallelism or K2 overlap.
 * A scheduler knob: batching trades each turn's time to first token for
 * throughput (GEMMs over thousands of rows instead of a few hundred). */
int askv_prefill_layers_batch(const askv_prefill_plan* plans, int njobs, void* stream);
/* Cumulative host microseconds of the layer loop's issue path since load:
 * out4 = {calls, capture (issuing the loop into the graph), update /
 * instantiate, launch}.  Diagnostics. */
void askv_issue_stats(double* out4);

/*
 * K5 — NCCL for the tensor-parallel all-reduce (C5), bound at run time
 * (libnccl.so.2).  unique_id writes the 128-byte ncclUniqueId rank 0 shares
 * with the group; comm_init builds this rank's communicator (collective over
 * the group); allreduce_bf16 sums `elems` bf16 values (send may equal recv) on
 * `stream`.  Replaces: nothing in the reference (PAPER.md:501 names NCCL only
 * for "synchronization of the parallel GPU workers").
 */
int askv_nccl_unique_id(void* out128);
int askv_nccl_comm_init(int nranks, int rank, const void* id128, void** comm);
int askv_nccl_comm_destroy(void* comm);
int askv_nccl_allreduce_bf16(const void* send, void* recv, int64_t elems, void* comm,
                             void* stream);
/* Write the device globaltimer (ns) to *dst (device memory) in stream order:
 * a timing mark that stays cheap while the host link is saturated. */
int askv_stamp(uint64_t* dst, void* stream);
/* sizeof(askv_prefill_plan), so FFI mirrors can check their struct layout. */
size_t askv_prefill_plan_size(void);
/* Time cuBLASLt's top candidate algorithms for y[n][m] = x[n][k] W[m][k]^T at
 * n = 32, 64, ..., 1024, then every 512 up to n_max (scratch operands, on
 * `stream`, synchronising), and make the layer loop use each n bucket's
 * fastest one.  Optional; call once per projection shape before serving. */
int askv_gemm_autotune(int m, int k, int n_max, size_t workspace_bytes, void* stream);
/* The layer loop's projection GEMM on its own: y[n][m] (+)= x[n][k] W[m][k]^T,
 * bf16 in / out, fp32 accumulate, cuBLASLt with the tuned (or heuristic)
 * algorithm of the n bucket; `accumulate` adds into y (the residual). */
int askv_gemm(const void* x, const void* w, void* y, int n, int m, int k, int accumulate,
              void* workspace, size_t workspace_bytes, void* stream);
/* Set the device's persisting-L2 set-aside (clamped to the device maximum) so
 * the evict_last hints on the layer's rotated K/V rows (K2 / rope_new stores,
 * K3 loads) can hold them in L2 between producer and consumer; *applied (may
 * be NULL) receives the size the driver set. */
int askv_l2_persist(size_t bytes, size_t* applied);

#ifdef __cplusplus
}
#endif
#endif /* ASKV_H_ */
