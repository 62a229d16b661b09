// RoPE-side kernels of the KV-reuse prefill path (sm_100a).
//
//   askv_rope_table : fp64-derived cos/sin table           (rope.py:55-60, 67-68)
//   askv_reembed    : K2 gather + truncate + re-embed       (rope.py:48-52, 63-74, 138;
//                                                            sim.py:468-483)
//   askv_rope_new   : new-token q/k rotation + pre-RoPE save copy (rope.py:139-140;
//                                                            PAPER.md:416-420)
//
// All three are HBM-bound elementwise kernels: each thread moves one 16-byte
// vector (8 bf16 = 4 interleaved rotation pairs), loads are read-only
// non-allocating, and the grid is a multiple of the SM count with a
// grid-stride loop.  The cos/sin table (<= a few MB) stays L2-resident.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "askv_internal.h"

namespace askv {
namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ int4 ld_nc16(const void* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
// Read-once load that asks L2 to evict the line first (K2's source rows must
// not displace the rotated rows it writes for K3).
__device__ __forceinline__ int4 ld_nc16_ef(const void* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void st16(void* p, int4 v) {
  asm volatile("st.global.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}
// Store that asks L2 to keep the line (attention's K/V rows are read right after).
__device__ __forceinline__ void st16_keep(void* p, int4 v) {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol)
               : "memory");
}

// Rotate the 4 interleaved pairs of a 16-byte bf16 vector by table entries
// cs[0..7] = (cos0, sin0, cos1, sin1, ...).
__device__ __forceinline__ int4 rotate8(int4 x, const float* cs) {
  const float4 a = *reinterpret_cast<const float4*>(cs);
  const float4 b = *reinterpret_cast<const float4*>(cs + 4);
  const float c[4] = {a.x, a.z, b.x, b.z};
  const float s[4] = {a.y, a.w, b.y, b.w};
  uint32_t w[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    __nv_bfloat162 p = *reinterpret_cast<__nv_bfloat162*>(&w[k]);
    const float e = __bfloat162float(p.x), o = __bfloat162float(p.y);
    const float r0 = fmaf(e, c[k], -(o * s[k]));
    const float r1 = fmaf(e, s[k], o * c[k]);
    __nv_bfloat162 q = __floats2bfloat162_rn(r0, r1);
    w[k] = *reinterpret_cast<uint32_t*>(&q);
  }
  return make_int4((int)w[0], (int)w[1], (int)w[2], (int)w[3]);
}

__global__ void rope_table_kernel(float* __restrict__ table, int max_pos, int half,
                                  double theta_base, int head_dim) {
  const int64_t total = (int64_t)max_pos * half;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int p = (int)(g / half);
    const int i = (int)(g - (int64_t)p * half);
    const double inv = pow(theta_base, -(2.0 * i) / (double)head_dim);
    double s, c;
    sincos((double)p * inv, &s, &c);
    table[2 * g] = (float)c;
    table[2 * g + 1] = (float)s;
  }
}

// K2: one CTA per `rows` consecutive rows (re_rows: 2 for wide K rows, up to
// kMaxReRows for GQA's narrow ones, ~1,000+ vectors per CTA).  The rows' cos/sin (rows x
// HD/2 float2) are staged in shared memory once, then every thread streams
// 16-byte vectors of the rows (4 in flight per thread), rotating K vectors
// and copying V vectors.  Source rows come through the session block table.
constexpr int kMaxReRows = 32;
// rows per CTA: two when a row's K is >= 512 16-byte vectors (13B: 640; four
// rows measured slower there), else enough rows for ~1,000 vectors (70B's
// 8 kv heads: 128 per row -> 8 rows), a power of two dividing the 128-row tile
inline int re_rows(int hkv, int head_dim) {
  const int units = hkv * head_dim / 8;
  if (units >= 512) return 2;
  int r = 2;
  while (r < kMaxReRows && (r * 2) * units <= 1280) r *= 2;
  return r;
}

// K2 over a batch of sessions in one launch (askv::reembed_batch): job i owns
// CTAs [cta0, next cta0) and its own block table / rows / destination; the
// source arena, row strides and RoPE table are shared.  n == 0: one job (the
// scalar arguments).
constexpr int kMaxReJobs = 24;
struct ReJobs {
  int n;
  int cta0[kMaxReJobs];
  int kept[kMaxReJobs];
  int v_from[kMaxReJobs];
  int pos0[kMaxReJobs];
  int64_t first_token[kMaxReJobs];
  const int64_t* blk_off[kMaxReJobs];
  __nv_bfloat16* dst[kMaxReJobs];
};

template <int HD>
__global__ void __launch_bounds__(kThreads)
    reembed_kernel(const __nv_bfloat16* __restrict__ src, const int64_t* __restrict__ blk_off,
                   int block_tokens, int64_t src_row_stride, int64_t first_token, int kept,
                   int hkv, const float* __restrict__ table, const int32_t* __restrict__ positions,
                   int pos0, __nv_bfloat16* __restrict__ dst, int64_t dst_row_stride,
                   unsigned long long* __restrict__ stamp, int v_from, int rows,
                   const __grid_constant__ ReJobs rj) {
  constexpr int kHalf = HD / 2;
  constexpr int kUnitsPerHead = HD / 8;
  // optional launch timestamps {begin of CTA 0, max CTA end} (attention.cu)
  if (stamp && threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamp[0] = t;
  }
  __shared__ __align__(16) float cs_s[kMaxReRows * kHalf * 2];
  __shared__ const __nv_bfloat16* srow_s[kMaxReRows];
  int row0 = blockIdx.x * rows;
  if (rj.n > 0) {  // batched: this CTA's job (positions are pos0 + row)
    int jb = 0;
    while (jb + 1 < rj.n && rj.cta0[jb + 1] <= (int)blockIdx.x) ++jb;
    row0 = (blockIdx.x - rj.cta0[jb]) * rows;
    blk_off = rj.blk_off[jb];
    first_token = rj.first_token[jb];
    kept = rj.kept[jb];
    pos0 = rj.pos0[jb];
    dst = rj.dst[jb];
    v_from = rj.v_from[jb];
  }
  const int nrows = min(rows, kept - row0);
  for (int i = threadIdx.x; i < nrows * kHalf; i += kThreads) {
    const int rr = i / kHalf, pi = i - rr * kHalf;
    const int pos = positions ? positions[row0 + rr] : pos0 + row0 + rr;
    const float2 v = reinterpret_cast<const float2*>(table)[(int64_t)pos * kHalf + pi];
    reinterpret_cast<float2*>(cs_s)[i] = v;
  }
  if (threadIdx.x < nrows) {
    const int64_t t = first_token + row0 + threadIdx.x;
    if (blk_off != nullptr) {
      const int64_t b = t / block_tokens;
      srow_s[threadIdx.x] = src + blk_off[b] + (t - b * block_tokens) * src_row_stride;
    } else {
      srow_s[threadIdx.x] = src + t * src_row_stride;
    }
  }
  __syncthreads();
  const int k_units = hkv * kUnitsPerHead;
  // rows below v_from: K only (their V is read by K3 straight from the
  // source); v_from is a multiple of the 128-row KV tile and `rows` a power of
  // two dividing it, so a CTA's rows are all on the same side of it
  const int row_units = row0 >= v_from ? 2 * k_units : k_units;
  const int total = nrows * row_units;
  // 13B: 2 rows x 640 K vectors = one round of 5 per thread; with two rows
  // the row of a vector is a compare, not an integer division (K2 was
  // issue-bound: ncu 45-50 % issue slots, profiles/r01d_summary.md)
  auto row_of = [&](int g) { return rows == 2 ? (g >= row_units ? 1 : 0) : g / row_units; };
  constexpr int kIlp = 5;
  const uint64_t pol_src = policy_evict_first();
  for (int base = threadIdx.x; base < total; base += kThreads * kIlp) {
    int4 v[kIlp];
#pragma unroll
    for (int k = 0; k < kIlp; ++k) {
      const int g = base + k * kThreads;
      if (g < total) {
        const int rr = row_of(g);
        v[k] = ld_nc16_ef(srow_s[rr] + (g - rr * row_units) * 8, pol_src);
      }
    }
#pragma unroll
    for (int k = 0; k < kIlp; ++k) {
      const int g = base + k * kThreads;
      if (g < total) {
        const int rr = row_of(g);
        const int u = g - rr * row_units;
        int4 x = v[k];
        if (u < k_units) x = rotate8(x, cs_s + (rr * kHalf + (u % kUnitsPerHead) * 4) * 2);
        st16_keep(dst + (int64_t)(row0 + rr) * dst_row_stride + u * 8, x);
      }
    }
  }
  if (stamp) {
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(stamp + 1, t);
    }
  }
}

// grid.y = new token, grid.x strides its 16-byte vectors (q heads, then K, V)
// with kRopeIlp loads in flight per thread.
constexpr int kRopeIlp = 4;

// Batched rope_new (askv_prefill_layers_batch): the jobs' new tokens are
// consecutive rows of qkv / q_out; token i of the launch belongs to the job
// with the last tok0 <= i, which has its own first position (its kept rows)
// and its own K|V and save destinations.  By value in the kernel parameters.
constexpr int kMaxRopeJobs = 24;
struct RopeJobs {
  int n;   // 0: one job (the scalar arguments)
  int tok0[kMaxRopeJobs];
  int pos0[kMaxRopeJobs];
  __nv_bfloat16* kv_out[kMaxRopeJobs];
  __nv_bfloat16* save_out[kMaxRopeJobs];
};

template <int HD>
__global__ void __launch_bounds__(kThreads)
    rope_new_kernel(const __nv_bfloat16* __restrict__ qkv, int64_t qkv_row_stride, int n_new,
                    int hq, int hkv, const float* __restrict__ table, int pos0,
                    __nv_bfloat16* __restrict__ q_out, __nv_bfloat16* __restrict__ kv_out,
                    int64_t kv_row_stride, __nv_bfloat16* __restrict__ save_out,
                    unsigned long long* __restrict__ end, const __grid_constant__ RopeJobs rj) {
  constexpr int kUnitsPerHead = HD / 8;
  const int q_units = hq * kUnitsPerHead;
  const int k_units = hkv * kUnitsPerHead;
  const int row_units = q_units + 2 * k_units;
  const int i = blockIdx.y;
  const __nv_bfloat16* src = qkv + (int64_t)i * qkv_row_stride;
  int li = i;   // the token's index within its job
  if (rj.n > 0) {
    int j = 0;
    while (j + 1 < rj.n && rj.tok0[j + 1] <= i) ++j;
    li = i - rj.tok0[j];
    pos0 = rj.pos0[j];
    kv_out = rj.kv_out[j];
    save_out = rj.save_out[j];
  }
  const float* cs_row = table + (int64_t)(pos0 + li) * HD;  // (cos, sin) x HD/2
  for (int u0 = blockIdx.x * kThreads * kRopeIlp + threadIdx.x; u0 < row_units;
       u0 += gridDim.x * kThreads * kRopeIlp) {
    int4 x[kRopeIlp];
#pragma unroll
    for (int k = 0; k < kRopeIlp; ++k) {
      const int u = u0 + k * kThreads;
      if (u < row_units) x[k] = ld_nc16(src + u * 8);
    }
#pragma unroll
    for (int k = 0; k < kRopeIlp; ++k) {
      const int u = u0 + k * kThreads;
      if (u >= row_units) break;
      const float* cs = cs_row + (u % kUnitsPerHead) * 8;
      if (u < q_units) {
        st16(q_out + (int64_t)i * q_units * 8 + u * 8, rotate8(x[k], cs));
      } else {
        const int ku = u - q_units;  // [0, 2*k_units): K then V, same as the row layout
        if (save_out != nullptr) st16(save_out + (int64_t)li * 2 * k_units * 8 + ku * 8, x[k]);
        st16_keep(kv_out + (int64_t)li * kv_row_stride + ku * 8,
                  ku < k_units ? rotate8(x[k], cs) : x[k]);
      }
    }
  }
  if (end) {  // timeline: latest CTA end (runtime.cu, the pre-load wait begins here)
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      atomicMax(end, t);
    }
  }
}

template <int HD>
__global__ void __launch_bounds__(kThreads)
    rotate_rows_kernel(const __nv_bfloat16* __restrict__ x, int64_t x_row_stride, int n_rows,
                       int heads, const float* __restrict__ table,
                       const int32_t* __restrict__ positions, int pos0,
                       __nv_bfloat16* __restrict__ out, int64_t out_row_stride) {
  constexpr int kUnitsPerHead = HD / 8;
  const int row_units = heads * kUnitsPerHead;
  const int64_t total = (int64_t)n_rows * row_units;
  for (int64_t g = blockIdx.x * (int64_t)kThreads + threadIdx.x; g < total;
       g += (int64_t)gridDim.x * kThreads) {
    const int i = (int)(g / row_units);
    const int u = (int)(g - (int64_t)i * row_units);
    const int pos = positions ? positions[i] : pos0 + i;
    const float* cs = table + ((int64_t)pos * (HD / 2) + (u % kUnitsPerHead) * 4) * 2;
    st16(out + (int64_t)i * out_row_stride + u * 8,
         rotate8(ld_nc16(x + (int64_t)i * x_row_stride + u * 8), cs));
  }
}

int grid_for(int64_t units) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (units + kThreads - 1) / kThreads;
  const int64_t cap = (int64_t)sms * 8;  // 8 x 256 threads resident per SM
  return (int)(want < cap ? (want > 0 ? want : 1) : cap);
}

}  // namespace
}  // namespace askv

using namespace askv;

extern "C" int askv_rope_table(float* table, int max_pos, int head_dim, double theta_base,
                               void* stream) {
  clear_error();
  ASKV_REQUIRE(table != nullptr, "rope_table: null table");
  ASKV_REQUIRE(max_pos > 0 && head_dim > 0 && head_dim % 2 == 0,
               "rope_table: bad max_pos=%d head_dim=%d (head_dim must be even)", max_pos,
               head_dim);
  const int half = head_dim / 2;
  const int64_t total = (int64_t)max_pos * half;
  int blocks = (int)((total + kThreads - 1) / kThreads);
  if (blocks > 4096) blocks = 4096;
  rope_table_kernel<<<blocks, kThreads, 0, (cudaStream_t)stream>>>(table, max_pos, half,
                                                                   theta_base, head_dim);
  return launch_status("rope_table launch");
}

extern "C" int askv_reembed(const void* src_base, const int64_t* src_block_off,
                            int block_tokens, int64_t src_row_stride, int64_t first_token,
                            int kept, int n_kv_heads, int head_dim, const float* rope_table,
                            int table_positions, const int32_t* positions, int pos0, void* dst,
                            int64_t dst_row_stride, void* stream) {
  clear_error();
  return askv::reembed_stamped(src_base, src_block_off, block_tokens, src_row_stride,
                               first_token, kept, n_kv_heads, head_dim, rope_table,
                               table_positions, positions, pos0, dst, dst_row_stride, stream,
                               nullptr, 0);
}

int askv::reembed_stamped(const void* src_base, const int64_t* src_block_off, int block_tokens,
                          int64_t src_row_stride, int64_t first_token, int kept, int n_kv_heads,
                          int head_dim, const float* rope_table, int table_positions,
                          const int32_t* positions, int pos0, void* dst, int64_t dst_row_stride,
                          void* stream, unsigned long long* stamp, int v_from) {
  ASKV_REQUIRE(kept >= 0 && n_kv_heads > 0 && first_token >= 0 && pos0 >= 0,
               "reembed: bad kept=%d hkv=%d first_token=%lld pos0=%d", kept, n_kv_heads,
               (long long)first_token, pos0);
  ASKV_REQUIRE(head_dim == 64 || head_dim == 128, "reembed: head_dim %d unsupported",
               head_dim);
  ASKV_REQUIRE(src_block_off == nullptr || block_tokens > 0, "reembed: block_tokens <= 0");
  ASKV_REQUIRE(positions != nullptr || pos0 + kept <= table_positions,
               "reembed: positions up to %d exceed rope table (%d)", pos0 + kept,
               table_positions);
  ASKV_REQUIRE(src_row_stride % 8 == 0 && dst_row_stride % 8 == 0,
               "reembed: row strides must be multiples of 8 elements");
  const int rows = re_rows(n_kv_heads, head_dim);
  ASKV_REQUIRE(v_from >= 0 && v_from % rows == 0,
               "reembed: v_from %d must be a multiple of %d rows", v_from, rows);
  if (kept == 0) return ASKV_OK;
  ASKV_REQUIRE(src_base && dst && rope_table, "reembed: null pointer");
  const int grid = (kept + rows - 1) / rows;
  auto* s = static_cast<const __nv_bfloat16*>(src_base);
  auto* d = static_cast<__nv_bfloat16*>(dst);
  ReJobs none;
  none.n = 0;
  if (head_dim == 128)
    reembed_kernel<128><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        s, src_block_off, block_tokens, src_row_stride, first_token, kept, n_kv_heads,
        rope_table, positions, pos0, d, dst_row_stride, stamp, v_from, rows, none);
  else
    reembed_kernel<64><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        s, src_block_off, block_tokens, src_row_stride, first_token, kept, n_kv_heads,
        rope_table, positions, pos0, d, dst_row_stride, stamp, v_from, rows, none);
  return launch_status("reembed launch");
}

int askv::reembed_batch(const void* src_base, int block_tokens, int64_t src_row_stride,
                        int n_jobs, const int64_t* const* blk_off, const int64_t* first_token,
                        const int* kept, const int* pos0, const int* v_from, void* const* dst,
                        int64_t dst_row_stride, int n_kv_heads, int head_dim,
                        const float* rope_table, int table_positions, void* stream,
                        unsigned long long* stamp) {
  ASKV_REQUIRE(n_jobs > 0 && n_kv_heads > 0 && block_tokens > 0,
               "reembed_batch: bad n_jobs=%d hkv=%d block_tokens=%d", n_jobs, n_kv_heads,
               block_tokens);
  ASKV_REQUIRE(head_dim == 64 || head_dim == 128, "reembed_batch: head_dim %d unsupported",
               head_dim);
  ASKV_REQUIRE(src_row_stride % 8 == 0 && dst_row_stride % 8 == 0,
               "reembed_batch: row strides must be multiples of 8 elements");
  ASKV_REQUIRE(src_base && rope_table, "reembed_batch: null pointer");
  auto* s = static_cast<const __nv_bfloat16*>(src_base);
  const int rows = re_rows(n_kv_heads, head_dim);
  for (int i0 = 0; i0 < n_jobs; i0 += kMaxReJobs) {
    ReJobs rj;
    rj.n = 0;
    int ctas = 0;
    for (int i = i0; i < n_jobs && i < i0 + kMaxReJobs; ++i) {
      if (kept[i] == 0) continue;
      ASKV_REQUIRE(kept[i] > 0 && first_token[i] >= 0 && pos0[i] >= 0 &&
                       pos0[i] + kept[i] <= table_positions && v_from[i] >= 0 &&
                       v_from[i] % rows == 0 && blk_off[i] && dst[i],
                   "reembed_batch: job %d (kept %d, pos0 %d, v_from %d)", i, kept[i], pos0[i],
                   v_from[i]);
      const int k = rj.n++;
      rj.cta0[k] = ctas;
      rj.kept[k] = kept[i];
      rj.v_from[k] = v_from[i];
      rj.pos0[k] = pos0[i];
      rj.first_token[k] = first_token[i];
      rj.blk_off[k] = blk_off[i];
      rj.dst[k] = static_cast<__nv_bfloat16*>(dst[i]);
      ctas += (kept[i] + rows - 1) / rows;
    }
    if (rj.n == 0) continue;
    // only the first launch of a batch carries the stamps
    unsigned long long* st = i0 == 0 ? stamp : nullptr;
    if (head_dim == 128)
      reembed_kernel<128><<<ctas, kThreads, 0, (cudaStream_t)stream>>>(
          s, nullptr, block_tokens, src_row_stride, 0, 0, n_kv_heads, rope_table, nullptr, 0,
          nullptr, dst_row_stride, st, 0, rows, rj);
    else
      reembed_kernel<64><<<ctas, kThreads, 0, (cudaStream_t)stream>>>(
          s, nullptr, block_tokens, src_row_stride, 0, 0, n_kv_heads, rope_table, nullptr, 0,
          nullptr, dst_row_stride, st, 0, rows, rj);
    const int rc = launch_status("reembed_batch launch");
    if (rc) return rc;
  }
  return ASKV_OK;
}

extern "C" int askv_rope_new(const void* qkv, int64_t qkv_row_stride, int n_new, int n_heads,
                             int n_kv_heads, int head_dim, const float* rope_table,
                             int table_positions, int pos0, void* q_out, void* kv_out,
                             int64_t kv_row_stride, void* save_out, void* stream) {
  clear_error();
  return askv::rope_new_stamped(qkv, qkv_row_stride, n_new, n_heads, n_kv_heads, head_dim,
                                rope_table, table_positions, pos0, q_out, kv_out, kv_row_stride,
                                save_out, stream, nullptr);
}

int askv::rope_new_stamped(const void* qkv, int64_t qkv_row_stride, int n_new, int n_heads,
                           int n_kv_heads, int head_dim, const float* rope_table,
                           int table_positions, int pos0, void* q_out, void* kv_out,
                           int64_t kv_row_stride, void* save_out, void* stream,
                           unsigned long long* end) {
  ASKV_REQUIRE(n_new >= 0 && n_heads > 0 && n_kv_heads > 0 && n_heads % n_kv_heads == 0,
               "rope_new: bad n_new=%d hq=%d hkv=%d", n_new, n_heads, n_kv_heads);
  ASKV_REQUIRE(head_dim == 64 || head_dim == 128, "rope_new: head_dim %d unsupported",
               head_dim);
  ASKV_REQUIRE(pos0 >= 0 && pos0 + n_new <= table_positions,
               "rope_new: positions up to %d exceed rope table (%d)", pos0 + n_new,
               table_positions);
  ASKV_REQUIRE(qkv_row_stride % 8 == 0 && kv_row_stride % 8 == 0,
               "rope_new: row strides must be multiples of 8 elements");
  if (n_new == 0) return ASKV_OK;
  ASKV_REQUIRE(qkv && q_out && kv_out && rope_table, "rope_new: null pointer");
  ASKV_REQUIRE(n_new <= 65535, "rope_new: %d new tokens exceed the grid's y limit", n_new);
  const int row_units = (n_heads + 2 * n_kv_heads) * (head_dim / 8);
  const dim3 grid((row_units + kThreads * kRopeIlp - 1) / (kThreads * kRopeIlp), n_new);
  auto* x = static_cast<const __nv_bfloat16*>(qkv);
  auto* qo = static_cast<__nv_bfloat16*>(q_out);
  auto* kvo = static_cast<__nv_bfloat16*>(kv_out);
  auto* so = static_cast<__nv_bfloat16*>(save_out);
  RopeJobs one;
  one.n = 0;
  if (head_dim == 128)
    rope_new_kernel<128><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        x, qkv_row_stride, n_new, n_heads, n_kv_heads, rope_table, pos0, qo, kvo,
        kv_row_stride, so, end, one);
  else
    rope_new_kernel<64><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        x, qkv_row_stride, n_new, n_heads, n_kv_heads, rope_table, pos0, qo, kvo,
        kv_row_stride, so, end, one);
  return launch_status("rope_new launch");
}

int askv::rope_new_batch(const void* qkv, int64_t qkv_row_stride, int n_jobs, const int* n_new,
                         const int* pos0, int n_heads, int n_kv_heads, int head_dim,
                         const float* rope_table, int table_positions, void* q_out,
                         void* const* kv_out, int64_t kv_row_stride, void* const* save_out,
                         void* stream, unsigned long long* end) {
  ASKV_REQUIRE(n_jobs >= 1 && n_heads > 0 && n_kv_heads > 0 && n_heads % n_kv_heads == 0,
               "rope_new_batch: bad jobs=%d hq=%d hkv=%d", n_jobs, n_heads, n_kv_heads);
  ASKV_REQUIRE(head_dim == 64 || head_dim == 128, "rope_new_batch: head_dim %d", head_dim);
  const int row_units = (n_heads + 2 * n_kv_heads) * (head_dim / 8);
  const int64_t q_stride_el = (int64_t)n_heads * head_dim;
  int tok = 0;
  for (int i0 = 0; i0 < n_jobs; i0 += kMaxRopeJobs) {   // <= kMaxRopeJobs jobs per launch
    RopeJobs rj;
    rj.n = n_jobs - i0 < kMaxRopeJobs ? n_jobs - i0 : kMaxRopeJobs;
    int tokens = 0;
    for (int k = 0; k < rj.n; ++k) {
      const int i = i0 + k;
      ASKV_REQUIRE(n_new[i] > 0 && pos0[i] >= 0 && pos0[i] + n_new[i] <= table_positions &&
                       kv_out[i],
                   "rope_new_batch: job %d (n_new %d, pos0 %d, table %d)", i, n_new[i], pos0[i],
                   table_positions);
      rj.tok0[k] = tokens;
      rj.pos0[k] = pos0[i];
      rj.kv_out[k] = static_cast<__nv_bfloat16*>(kv_out[i]);
      rj.save_out[k] = save_out ? static_cast<__nv_bfloat16*>(save_out[i]) : nullptr;
      tokens += n_new[i];
    }
    ASKV_REQUIRE(tokens <= 65535, "rope_new_batch: %d tokens exceed the grid's y limit", tokens);
    const dim3 grid((row_units + kThreads * kRopeIlp - 1) / (kThreads * kRopeIlp), tokens);
    auto* x = static_cast<const __nv_bfloat16*>(qkv) + (int64_t)tok * qkv_row_stride;
    auto* qo = static_cast<__nv_bfloat16*>(q_out) + (int64_t)tok * q_stride_el;
    if (head_dim == 128)
      rope_new_kernel<128><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
          x, qkv_row_stride, tokens, n_heads, n_kv_heads, rope_table, 0, qo, nullptr,
          kv_row_stride, nullptr, end, rj);
    else
      rope_new_kernel<64><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
          x, qkv_row_stride, tokens, n_heads, n_kv_heads, rope_table, 0, qo, nullptr,
          kv_row_stride, nullptr, end, rj);
    const int rc = launch_status("rope_new_batch launch");
    if (rc) return rc;
    tok += tokens;
  }
  return ASKV_OK;
}

extern "C" int askv_rotate_rows(const void* x, int64_t x_row_stride, int n_rows, int n_heads,
                                int head_dim, const float* rope_table, int table_positions,
                                const int32_t* positions, int pos0, void* out,
                                int64_t out_row_stride, void* stream) {
  clear_error();
  ASKV_REQUIRE(n_rows >= 0 && n_heads > 0, "rotate_rows: bad n_rows=%d heads=%d", n_rows,
               n_heads);
  ASKV_REQUIRE(head_dim == 64 || head_dim == 128, "rotate_rows: head_dim %d unsupported",
               head_dim);
  ASKV_REQUIRE(positions != nullptr || (pos0 >= 0 && pos0 + n_rows <= table_positions),
               "rotate_rows: positions up to %d exceed rope table (%d)", pos0 + n_rows,
               table_positions);
  ASKV_REQUIRE(x_row_stride % 8 == 0 && out_row_stride % 8 == 0,
               "rotate_rows: row strides must be multiples of 8 elements");
  if (n_rows == 0) return ASKV_OK;
  ASKV_REQUIRE(x && out && rope_table, "rotate_rows: null pointer");
  const int grid = grid_for((int64_t)n_rows * n_heads * (head_dim / 8));
  auto* xi = static_cast<const __nv_bfloat16*>(x);
  auto* o = static_cast<__nv_bfloat16*>(out);
  if (head_dim == 128)
    rotate_rows_kernel<128><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        xi, x_row_stride, n_rows, n_heads, rope_table, positions, pos0, o, out_row_stride);
  else
    rotate_rows_kernel<64><<<grid, kThreads, 0, (cudaStream_t)stream>>>(
        xi, x_row_stride, n_rows, n_heads, rope_table, positions, pos0, o, out_row_stride);
  return launch_status("rotate_rows launch");
}
