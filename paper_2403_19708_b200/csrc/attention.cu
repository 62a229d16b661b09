// K3 — prefill attention over [reused prefix | new tokens] on sm_100a.
//
// Semantics (rope.py:94-105 inside rope.py:118-144): out = softmax(q k^T / sqrt(d)) v
// where query i (0-based among the n_new new tokens) sees key rows
// j <= n_cached + i.  q and k arrive already rotated (K2 / rope_new).
//
// One CTA = one 128-row query tile x one q-head x one KV split.  Warp roles:
//   warp 0      TMA producer: Q once, then K/V 128-row tiles into a STAGES ring
//   warp 1      MMA issuer (one thread): S = Q K^T into a double-buffered TMEM
//               tile, then O_j = P_j V_j into a TMEM tile (tcgen05.mma kind::f16)
//   warp 2      TMEM allocator (512 columns: S0 | S1 | O)
//   warps 4-7   softmax: thread r owns query row r (= TMEM lane r); reads S with
//               tcgen05.ld, online softmax in fp32 (exp2), writes P (bf16) into a
//               SWIZZLE_128B K-major smem tile for the PV MMA, folds each
//               finished O_j into a register accumulator with the running-max
//               correction, and writes the normalised row (or a split partial).
// The MMA warp issues S_{j+1} before PV_j, so QK^T of the next tile runs on the
// tensor core while the softmax warps work on the current one.
//
// Layouts: Q [n_new][Hq][d]; K/V rows [T][2][Hkv][d] (token-major, K then V,
// exactly the host-block row layout so preloaded blocks are used in place);
// tiles are fetched by 3-D TMA maps {d, head, row} with 64-element (128 B)
// boxes and SWIZZLE_128B, which is the canonical UMMA K-major layout for Q/K
// and MN-major layout for V (B operand of PV).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <mutex>

#include "askv_internal.h"
#include "askv_ptx.cuh"

namespace askv {
namespace {

constexpr int kBM = 128;  // query rows per tile (UMMA M)
constexpr int kBN = 128;  // key rows per tile (UMMA N of S, K of PV)
constexpr int kThreads = 256;
constexpr int kMaxSplits = 32;

template <int HD>
struct Cfg {
  static constexpr int kStages = HD == 128 ? 2 : 4;
  static constexpr int kChunks = HD / 64;                  // 64-col swizzle chunks
  static constexpr int kTileBytes = kBM * HD * 2;          // Q / K / V tile
  static constexpr int kPBytes = kBM * kBN * 2;            // P tile
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + kTileBytes;
  static constexpr int kVOff = kKOff + kStages * kTileBytes;
  static constexpr int kPOff = kVOff + kStages * kTileBytes;
  static constexpr int kBarOff = kPOff + kPBytes;
  // barriers: q_full, k_full[S], v_full[S], kv_empty[S], s_full[2], s_empty[2],
  //           p_full, o_full, o_empty
  static constexpr int kNumBars = 1 + 3 * kStages + 4 + 3;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kSmemBytes = kTmemSlotOff + 16 + 1024;  // +1024 manual alignment
  static constexpr uint32_t kTmemCols = 512;
  static constexpr uint32_t kColS0 = 0, kColS1 = 128, kColO = 256;
};

struct AttnParams {
  int n_new;
  int n_cached;
  int hq;
  int group;
  int num_splits;
  int tiles_per_split;
  float scale_log2;
  __nv_bfloat16* out;  // [n_new][hq][HD]
  float* part_o;       // [splits][n_new][hq][HD]
  float* part_lse;     // [splits][n_new][hq]   (log2 units)
};

template <int HD>
__global__ void __launch_bounds__(kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v, const AttnParams p) {
  using C = Cfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sK = smem + C::kKOff;
  uint8_t* sV = smem + C::kVOff;
  uint8_t* sP = smem + C::kPOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* v_full = k_full + C::kStages;
  uint64_t* kv_empty = v_full + C::kStages;
  uint64_t* s_full = kv_empty + C::kStages;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* o_full = p_full + 1;
  uint64_t* o_empty = o_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kTmemSlotOff);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x;
  const int h = blockIdx.y;
  const int split = blockIdx.z;
  const int kh = h / p.group;
  const int q0 = m_tile * kBM;
  const int q_rows = min(kBM, p.n_new - q0);
  const int kv_end = p.n_cached + q0 + q_rows;  // exclusive
  const int tiles_total = (kv_end + kBN - 1) / kBN;
  const int t_begin = split * p.tiles_per_split;
  const int t_end = min(tiles_total, t_begin + p.tiles_per_split);
  const int n_tiles = t_end > t_begin ? t_end - t_begin : 0;
  const bool partial = p.num_splits > 1;

  if (n_tiles == 0) {  // empty split: neutral partial (CTA-uniform branch)
    if (warp >= 4) {
      const int r = threadIdx.x - 128;
      const int qi = q0 + r;
      if (r < q_rows) {
        const int64_t row = ((int64_t)split * p.n_new + qi) * p.hq + h;
        p.part_lse[row] = -INFINITY;
        float4* po = reinterpret_cast<float4*>(p.part_o + row * HD);
#pragma unroll
        for (int c = 0; c < HD / 4; ++c) po[c] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    return;
  }

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&kv_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&s_full[b], 1);
      mbar_init(&s_empty[b], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    mbar_init(o_empty, 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      mbar_expect_tx(q_full, C::kTileBytes);
#pragma unroll
      for (int c = 0; c < C::kChunks; ++c)
        tma_load_3d(sQ + c * (kBM * 128), &tm_q, q_full, c * 64, h, q0);
      for (int j = 0; j < n_tiles; ++j) {
        const int st = j % C::kStages;
        if (j >= C::kStages) mbar_wait(&kv_empty[st], ((j / C::kStages) - 1) & 1);
        const int row0 = (t_begin + j) * kBN;
        uint8_t* dk = sK + st * C::kTileBytes;
        uint8_t* dv = sV + st * C::kTileBytes;
        mbar_expect_tx(&k_full[st], C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dk + c * (kBN * 128), &tm_k, &k_full[st], c * 64, kh, row0);
        mbar_expect_tx(&v_full[st], C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d(dv + c * (kBN * 128), &tm_v, &v_full[st], c * 64, kh, row0);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kBM, kBN, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kBM, HD, 0, 1);
      const uint32_t sq = smem_u32(sQ), sk = smem_u32(sK), sv = smem_u32(sV),
                     sp = smem_u32(sP);
      mbar_wait(q_full, 0);
      auto issue_s = [&](int j) {
        const int st = j % C::kStages;
        const int b = j & 1;
        mbar_wait(&k_full[st], (j / C::kStages) & 1);
        if (j >= 2) mbar_wait(&s_empty[b], ((j >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + (b ? C::kColS1 : C::kColS0);
        const uint32_t kb = sk + st * C::kTileBytes;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = (k >> 2) * (kBM * 128) + (k & 3) * 32;
          umma_bf16(d, sdesc_sw128(sq + off, 16, 1024), sdesc_sw128(kb + off, 16, 1024),
                    idesc_s, k > 0);
        }
        umma_commit(&s_full[b]);
      };
      issue_s(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) issue_s(j + 1);
        const int st = j % C::kStages;
        mbar_wait(p_full, j & 1);
        mbar_wait(&v_full[st], (j / C::kStages) & 1);
        if (j >= 1) mbar_wait(o_empty, (j - 1) & 1);
        tc_fence_after();
        const uint32_t vb = sv + st * C::kTileBytes;
#pragma unroll
        for (int k = 0; k < kBN / 16; ++k) {
          const uint32_t aoff = (k >> 2) * (kBM * 128) + (k & 3) * 32;
          umma_bf16(tmem + C::kColO, sdesc_sw128(sp + aoff, 16, 1024),
                    sdesc_sw128(vb + k * (16 * 128), kBN * 128, 1024), idesc_o, k > 0);
        }
        umma_commit(o_full);
        umma_commit(&kv_empty[st]);
      }
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    const int r = threadIdx.x - 128;  // row in tile == TMEM lane
    const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
    const int qi = q0 + r;
    const int row_limit = p.n_cached + qi;  // last visible key
    const float sl2 = p.scale_log2;
    float o[HD];
#pragma unroll
    for (int c = 0; c < HD; ++c) o[c] = 0.f;
    float m_acc = -INFINITY, l_acc = 0.f;  // accumulator state
    float m_run = -INFINITY;               // running max (scaled, log2 units)
    float m_prev = -INFINITY, l_prev = 0.f;  // stats of the in-flight PV tile
    uint8_t* prow = sP + r * 128;
    const int sw = r & 7;

    // Fold PV_j (relative to m_prev) into the register accumulator.  The
    // tcgen05.ld calls are warp-collective, so the per-row "tile fully masked"
    // case is handled with coefficients, not a branch.
    auto fold = [&](int j) {
      mbar_wait(o_full, j & 1);
      tc_fence_after();
      float a_o = 1.f, b_pv = 0.f;
      if (m_prev != -INFINITY) {
        a_o = (m_acc == -INFINITY) ? 0.f : ex2(m_acc - m_prev);
        b_pv = 1.f;
        l_acc = l_acc * a_o + l_prev;
        m_acc = m_prev;
      }
#pragma unroll
      for (int c = 0; c < HD / 32; ++c) {
        float pv[32];
        tmem_ld32(trow + C::kColO + c * 32, pv);
#pragma unroll
        for (int e = 0; e < 32; ++e) o[c * 32 + e] = fmaf(pv[e], b_pv, o[c * 32 + e] * a_o);
      }
    };

    for (int j = 0; j < n_tiles; ++j) {
      const int b = j & 1;
      const uint32_t scol = b ? C::kColS1 : C::kColS0;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_fence_after();
      const int kbase = (t_begin + j) * kBN;
      const int lim = row_limit - kbase;  // columns c <= lim are visible
      float mx = -INFINITY;
#pragma unroll
      for (int c = 0; c < kBN / 32; ++c) {
        float s[32];
        tmem_ld32(trow + scol + c * 32, s);
#pragma unroll
        for (int e = 0; e < 32; ++e) mx = fmaxf(mx, (c * 32 + e <= lim) ? s[e] : -INFINITY);
      }
      const float m_new = fmaxf(m_run, mx * sl2);
      if (j >= 1) {
        fold(j - 1);
        tc_fence_before();
        mbar_arrive(o_empty);
      }
      // P_j = exp2(S * scale_log2 - m_new), bf16, into the swizzled K-major tile
      float lsum = 0.f;
      const float neg_m = (m_new == -INFINITY) ? 0.f : -m_new;
#pragma unroll
      for (int c = 0; c < kBN / 32; ++c) {
        float s[32];
        tmem_ld32(trow + scol + c * 32, s);
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float p0 = (c * 32 + e <= lim) ? ex2(fmaf(s[e], sl2, neg_m)) : 0.f;
          const float p1 = (c * 32 + e + 1 <= lim) ? ex2(fmaf(s[e + 1], sl2, neg_m)) : 0.f;
          lsum += p0 + p1;
          pk[e >> 1] = pack_bf16x2(p0, p1);
        }
        uint8_t* half = prow + (c >> 1) * (kBM * 128);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
          const int u = (c & 1) * 4 + w;
          *reinterpret_cast<uint4*>(half + ((u ^ sw) << 4)) =
              make_uint4(pk[4 * w], pk[4 * w + 1], pk[4 * w + 2], pk[4 * w + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&s_empty[b]);
      fence_proxy_async_smem();
      mbar_arrive(p_full);
      m_prev = m_new;
      l_prev = lsum;
      m_run = m_new;
    }
    fold(n_tiles - 1);
    tc_fence_before();

    if (r < q_rows) {
      const float inv_l = l_acc > 0.f ? 1.f / l_acc : 0.f;
      if (!partial) {
        __nv_bfloat16* dst = p.out + ((int64_t)qi * p.hq + h) * HD;
#pragma unroll
        for (int c = 0; c < HD / 8; ++c) {
          uint4 v;
          v.x = pack_bf16x2(o[8 * c + 0] * inv_l, o[8 * c + 1] * inv_l);
          v.y = pack_bf16x2(o[8 * c + 2] * inv_l, o[8 * c + 3] * inv_l);
          v.z = pack_bf16x2(o[8 * c + 4] * inv_l, o[8 * c + 5] * inv_l);
          v.w = pack_bf16x2(o[8 * c + 6] * inv_l, o[8 * c + 7] * inv_l);
          reinterpret_cast<uint4*>(dst)[c] = v;
        }
      } else {
        const int64_t row = ((int64_t)split * p.n_new + qi) * p.hq + h;
        p.part_lse[row] = l_acc > 0.f ? m_acc + __log2f(l_acc) : -INFINITY;
        float4* po = reinterpret_cast<float4*>(p.part_o + row * HD);
#pragma unroll
        for (int c = 0; c < HD / 4; ++c)
          po[c] = make_float4(o[4 * c] * inv_l, o[4 * c + 1] * inv_l, o[4 * c + 2] * inv_l,
                              o[4 * c + 3] * inv_l);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

// Deterministic split-KV combine: one warp per (query, head), splits in order.
template <int HD>
__global__ void __launch_bounds__(128)
    attn_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_lse,
                        int num_splits, int rows, __nv_bfloat16* __restrict__ out) {
  const int row = blockIdx.x * 4 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float m = -INFINITY;
  for (int s = 0; s < num_splits; ++s) m = fmaxf(m, part_lse[(int64_t)s * rows + row]);
  constexpr int kPer = HD / 32;
  float acc[kPer] = {};
  float wsum = 0.f;
  for (int s = 0; s < num_splits; ++s) {
    const float l = part_lse[(int64_t)s * rows + row];
    if (l == -INFINITY) continue;
    const float w = exp2f(l - m);
    wsum += w;
    const float* src = part_o + ((int64_t)s * rows + row) * HD + lane * kPer;
#pragma unroll
    for (int e = 0; e < kPer; ++e) acc[e] = fmaf(w, src[e], acc[e]);
  }
  const float inv = wsum > 0.f ? 1.f / wsum : 0.f;
  __nv_bfloat16* dst = out + (int64_t)row * HD + lane * kPer;
#pragma unroll
  for (int e = 0; e < kPer; e += 2)
    *reinterpret_cast<__nv_bfloat162*>(dst + e) =
        __floats2bfloat162_rn(acc[e] * inv, acc[e + 1] * inv);
}

// ---------------------------------------------------------------- host side
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                   const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                   const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion,
                                   CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(ptr);
  });
  return fn;
}

// 3-D bf16 map {d, heads, rows} with a {64, 1, 128} SWIZZLE_128B box.
int make_map(CUtensorMap* m, const void* base, int head_dim, int heads, int64_t head_stride,
             int64_t rows, int64_t row_stride) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ASKV_ECUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)head_dim, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)head_stride * 2, (cuuint64_t)row_stride * 2};
  cuuint32_t box[3] = {64, 1, 128};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", (int)r);
    return ASKV_ECUDA;
  }
  return ASKV_OK;
}

int sm_count() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// Split count minimising waves x (tiles per split + fixed per-CTA overhead).
int choose_splits(int n_cached, int n_new, int hq, int sms) {
  const int q_tiles = (n_new + kBM - 1) / kBM;
  const int kv_tiles = (n_cached + n_new + kBN - 1) / kBN;
  const int ctas = q_tiles * hq;
  int best = 1;
  double best_cost = 1e30;
  for (int s = 1; s <= kMaxSplits && s <= kv_tiles; ++s) {
    const int tps = (kv_tiles + s - 1) / s;
    const int eff = (kv_tiles + tps - 1) / tps;
    if (eff != s) continue;
    const int waves = (ctas * s + sms - 1) / sms;
    const double cost = waves * (tps + 1.5) + (s > 1 ? 0.3 : 0.0);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = s;
    }
  }
  return best;
}

template <int HD>
int launch_attn(const void* q, const void* kv, int64_t kv_row_stride, int n_cached, int n_new,
                int hq, int hkv, float scale, void* out, void* ws, size_t ws_bytes,
                int splits, cudaStream_t stream) {
  using C = Cfg<HD>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(attn_fwd_kernel<HD>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return cuda_status(e, "attn smem attribute");
    attr_set = true;
  }
  const int rows = n_cached + n_new;
  CUtensorMap mq, mk, mv;
  int rc = make_map(&mq, q, HD, hq, HD, n_new, (int64_t)hq * HD);
  if (!rc) rc = make_map(&mk, kv, HD, hkv, HD, rows, kv_row_stride);
  if (!rc)
    rc = make_map(&mv, static_cast<const __nv_bfloat16*>(kv) + (int64_t)hkv * HD, HD, hkv, HD,
                  rows, kv_row_stride);
  if (rc) return rc;

  const int q_tiles = (n_new + kBM - 1) / kBM;
  const int kv_tiles = (rows + kBN - 1) / kBN;
  const int tps = (kv_tiles + splits - 1) / splits;
  splits = (kv_tiles + tps - 1) / tps;
  AttnParams prm;
  prm.n_new = n_new;
  prm.n_cached = n_cached;
  prm.hq = hq;
  prm.group = hq / hkv;
  prm.num_splits = splits;
  prm.tiles_per_split = tps;
  prm.scale_log2 = scale * 1.4426950408889634f;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.part_o = nullptr;
  prm.part_lse = nullptr;
  if (splits > 1) {
    const size_t rows_qh = (size_t)n_new * hq;
    const size_t need = (size_t)splits * rows_qh * (HD + 1) * sizeof(float);
    ASKV_REQUIRE(ws != nullptr && ws_bytes >= need,
                 "prefill_attn: workspace %zu bytes < %zu needed for %d splits", ws_bytes, need,
                 splits);
    prm.part_o = static_cast<float*>(ws);
    prm.part_lse = prm.part_o + (size_t)splits * rows_qh * HD;
  }
  dim3 grid(q_tiles, hq, splits);
  attn_fwd_kernel<HD><<<grid, kThreads, C::kSmemBytes, stream>>>(mq, mk, mv, prm);
  rc = launch_status("attn_fwd launch");
  if (rc || splits == 1) return rc;
  const int rows_qh = n_new * hq;
  attn_combine_kernel<HD><<<(rows_qh + 3) / 4, 128, 0, stream>>>(
      prm.part_o, prm.part_lse, splits, rows_qh, static_cast<__nv_bfloat16*>(out));
  return launch_status("attn_combine launch");
}

}  // namespace
}  // namespace askv

using namespace askv;

extern "C" int askv_attn_num_splits(int n_cached, int n_new, int n_heads, int sms) {
  if (n_new <= 0 || n_heads <= 0 || n_cached < 0) return 1;
  return choose_splits(n_cached, n_new, n_heads, sms > 0 ? sms : sm_count());
}

extern "C" size_t askv_attn_workspace_bytes(int n_cached, int n_new, int n_heads,
                                            int head_dim, int num_splits) {
  if (n_new <= 0 || n_heads <= 0) return 0;
  const int s = num_splits > 0 ? num_splits : choose_splits(n_cached, n_new, n_heads, sm_count());
  if (s <= 1) return 0;
  return (size_t)s * n_new * n_heads * (head_dim + 1) * sizeof(float);
}

extern "C" int askv_prefill_attn(const void* q, const void* kv, int64_t kv_row_stride,
                                 int n_cached, int n_new, int n_heads, int n_kv_heads,
                                 int head_dim, float scale, void* out, void* workspace,
                                 size_t workspace_bytes, int num_splits, void* stream) {
  clear_error();
  ASKV_REQUIRE(n_cached >= 0 && n_new >= 0, "prefill_attn: negative lengths");
  ASKV_REQUIRE(n_heads > 0 && n_kv_heads > 0 && n_heads % n_kv_heads == 0,
               "prefill_attn: Hq=%d must be a positive multiple of Hkv=%d", n_heads,
               n_kv_heads);
  ASKV_REQUIRE(head_dim == 64 || head_dim == 128,
               "prefill_attn: head_dim %d unsupported (64, 128)", head_dim);
  ASKV_REQUIRE(num_splits >= 0 && num_splits <= kMaxSplits, "prefill_attn: bad num_splits");
  if (n_new == 0) return ASKV_OK;
  ASKV_REQUIRE(q && kv && out, "prefill_attn: null pointer");
  ASKV_REQUIRE(((uintptr_t)q & 15) == 0 && ((uintptr_t)kv & 15) == 0 && kv_row_stride % 8 == 0,
               "prefill_attn: q/kv must be 16-byte aligned with row stride %% 8 == 0");
  ASKV_REQUIRE(kv_row_stride >= 2LL * n_kv_heads * head_dim,
               "prefill_attn: kv_row_stride %lld < 2*Hkv*d", (long long)kv_row_stride);
  int splits = num_splits > 0 ? num_splits : choose_splits(n_cached, n_new, n_heads, sm_count());
  if (head_dim == 128)
    return launch_attn<128>(q, kv, kv_row_stride, n_cached, n_new, n_heads, n_kv_heads, scale,
                            out, workspace, workspace_bytes, splits, (cudaStream_t)stream);
  return launch_attn<64>(q, kv, kv_row_stride, n_cached, n_new, n_heads, n_kv_heads, scale, out,
                         workspace, workspace_bytes, splits, (cudaStream_t)stream);
}
