// K3 — prefill attention over [reused prefix | new tokens] on sm_100a.
//
// Semantics (rope.py:94-105 inside rope.py:118-144): out = softmax(q k^T / sqrt(d)) v
// where query i (0-based among the n_new new tokens) sees key rows
// j <= n_cached + i.  q and k arrive already rotated (K2 / rope_new).
//
// Design (kernel comment below): per CTA one 128-row query tile x one q-head x
// one KV split; two softmax warpgroups take alternate KV tiles and ping-pong
// on the tensor core; S, P and O live in TMEM; K/V stream through 3-deep TMA
// rings; split-KV partials merge in a deterministic combine kernel.
//
// Layouts: Q [n_new][Hq][d]; K/V rows [T][2][Hkv][d] (token-major, K then V,
// exactly the host-block row layout so preloaded blocks are used in place);
// tiles are fetched by 3-D TMA maps {d, head, row} with 64-element (128 B)
// boxes and SWIZZLE_128B, which is the canonical UMMA K-major layout for Q/K
// and MN-major layout for V (B operand of PV).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <map>
#include <mutex>
#include <type_traits>

#include "askv_internal.h"
#include "askv_ptx.cuh"

namespace askv {
namespace {

// Optional in-kernel timeline (tools/attn_trace.cu builds with ASKV_ATTN_TRACE):
// globaltimer stamps per CTA at fixed slots (256 per CTA; 192..255: phases of
// the softmax tile of WG0's thread 0, tiles 2..17).
#ifdef ASKV_ATTN_TRACE
__device__ unsigned long long* g_attn_trace = nullptr;
__device__ __forceinline__ void trace_stamp(int slot) {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  const int cta = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
  if (g_attn_trace) {
    g_attn_trace[cta * 256 + slot] = t;
    if (slot == 0) {
      unsigned sm;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
      g_attn_trace[cta * 256 + 5] = sm;  // slot 5: SM id
      g_attn_trace[cta * 256 + 6] = clock64();  // slots 6 / 7: SM clock at entry / exit
    }
    if (slot == 4) g_attn_trace[cta * 256 + 7] = clock64();
  }
}
#define ATTN_TRACE(slot) trace_stamp(slot)
#else
#define ATTN_TRACE(slot) ((void)0)
#endif

// Launch timestamps without extra launches (bench probes, plan.stamps):
// stamp[0] = globaltimer at the start of CTA (0,0,0) -- the first wave starts
// together -- and stamp[1] = max over CTAs of their end time (atomicMax; the
// ring slot's stale value is an older, smaller time, so no reset is needed).
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void launch_stamp_begin(unsigned long long* st) {
  if (st && threadIdx.x == 0 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
    st[0] = gtimer();
}
__device__ __forceinline__ void launch_stamp_end(unsigned long long* st) {
  if (st && threadIdx.x == 0) atomicMax(st + 1, gtimer());
}

// Quarters of the softmax exponentials evaluated on the FMA pipe (packed
// cubic) instead of MUFU ex2 (build-time A/B knob; 1 = one quarter), or an
// explicit mask over the 8 pair slots of each 16 columns (ASKV_ATTN_POLY_MASK).
#ifndef ASKV_ATTN_POLY_Q
#define ASKV_ATTN_POLY_Q 1
#endif
#ifndef ASKV_ATTN_POLY_MASK
#define ASKV_ATTN_POLY_MASK (0x11 * ((0xF0 >> ASKV_ATTN_POLY_Q) & 0xF))
#endif
// 1: off-diagonal tiles after a group's first skip the max pass (exps
// against the running max, overflow past the lazy threshold detected from
// the row sum / the polynomial lanes' max).  Same values as the max-first
// order; +5.7 % on the batched pass's varlen launch (attn_varlen_trace, two
// A/B pairs), neutral at single-launch shapes (attn_ab).  Build-time knob.
#ifndef ASKV_ATTN_SUMCHECK
#define ASKV_ATTN_SUMCHECK 1
#endif
#ifndef ASKV_ATTN_ELECT_ISSUE  // MMA warp: warp-converged issue, lane elected in the asm
#define ASKV_ATTN_ELECT_ISSUE 1
#endif
#ifndef ASKV_ATTN_INTERLEAVE  // paired: S_A(j+1) interleaved with PV_B(j) (A/B knob)
#define ASKV_ATTN_INTERLEAVE 0
#endif
#ifndef ASKV_ATTN_EARLY_VFREE  // paired: release a V slot right after its last PV
#define ASKV_ATTN_EARLY_VFREE 1
#endif
#ifndef ASKV_ATTN_PROBE  // pipeline probes, experiment builds only (see tile())
#define ASKV_ATTN_PROBE 0
#endif

constexpr int kBM = 128;  // query rows per tile (UMMA M)
constexpr int kBN = 128;  // key rows per tile (UMMA N of S, K of PV)
constexpr int kMaxSplits = 32;
constexpr int kMaxSkSlots = 24;  // stream-K: pieces per unit (combine smem)

struct AttnParams {
  int n_new;
  int n_cached;
  int hq;
  int group;
  int pack;  // > 1: GQA packing -- a CTA's 128 rows are (token, q-head) pairs of one kv head
  int num_splits;
  int tiles_per_split;
  float scale_log2;
  __nv_bfloat16* out;  // [n_new][hq][HD]
  unsigned long long* stamp;  // optional {begin, end} launch timestamps
  float* part_o;       // [splits][n_new][hq][HD]
  float* part_lse;     // [splits][n_new][hq]   (log2 units)
  // stream-K schedule (attn_sk_kernel): the KV tiles of every unit (query tile,
  // head), head-major, form one list of sk_total tiles cut into gridDim.x equal
  // contiguous ranges, one per CTA (= per SM, one wave)
  int sk_total;        // G: sum over units of their KV tiles
  int sk_tiles_head;   // KV tiles of one head's units
  int sk_q_tiles;      // query tiles per head (unit = (head, query tile))
  int sk_units;        // units = heads x sk_q_tiles (partial slab stride)
  int* sk_cnt;         // per-unit arrival counters (zero between launches)
  // V source (VSource, askv_internal.h): tiles < v_src_tiles load V through
  // tm_vs at row v_blk_off ? v_blk_off[t] / v_row_elems + v_layer_row
  //                         : v_src_row0 + 128 t
  int v_src_tiles;
  int64_t v_src_row0;
  const int64_t* v_blk_off;
  int64_t v_row_elems;
  int64_t v_layer_row;
};

// Varlen launch (a batch of jobs in one K3 launch, askv_prefill_layers_batch):
// per job its sizes, where its rows sit in the shared Q / KV buffers, its
// output, its V-source block table, and the first CTA of its (query tile,
// head) grid (1-D over all jobs).  Passed by value in the kernel parameters.
constexpr int kMaxVarJobs = 24;
struct VarJob {
  int n_new, n_cached, q_row0, kv_row0, cta0, q_groups, v_src_tiles;
  const int64_t* v_blk_off;
  int64_t v_layer_row;
  __nv_bfloat16* out;
};
struct VarJobs {
  int n;   // 0: not a varlen launch
  VarJob j[kMaxVarJobs];
};

// Where KV tile t's V rows come from: (use the V-source map?, row coordinate).
__device__ __forceinline__ int v_tile_row(const AttnParams& p, int t, bool& src) {
  src = t < p.v_src_tiles;
  if (!src) return t * kBN;
  return p.v_blk_off ? (int)(p.v_blk_off[t] / p.v_row_elems + p.v_layer_row)
                     : (int)(p.v_src_row0 + (int64_t)t * kBN);
}

// KV tiles query tile q must visit (keys <= n_cached + its last token).
__host__ __device__ __forceinline__ int unit_tiles(const AttnParams& p, int q) {
  const int q_rows = p.pack > 1 ? p.n_new * p.pack : p.n_new;
  const int last = (q + 1) * kBM < q_rows ? (q + 1) * kBM - 1 : q_rows - 1;
  const int tok = p.pack > 1 ? last / p.pack : last;
  return (p.n_cached + tok + 1 + kBN - 1) / kBN;
}

// One CTA's contiguous share of the stream-K tile list.
__host__ __device__ __forceinline__ void sk_range(const AttnParams& p, int c, int ctas, int& g0,
                                                  int& g1) {
  g0 = (int)((int64_t)c * p.sk_total / ctas);
  g1 = (int)((int64_t)(c + 1) * p.sk_total / ctas);
}

// CTA whose range holds global tile g.
__host__ __device__ __forceinline__ int sk_owner(const AttnParams& p, int g, int ctas) {
  return (int)(((int64_t)(g + 1) * ctas - 1) / p.sk_total);
}

// The piece of a unit that starts at global tile g inside [g, g1): which unit,
// its tile range, and the partial slot (CTA index relative to the unit's first
// CTA).  `whole` = the piece is the entire unit (final output, no combine).
struct Piece {
  int head, q, t_begin, t_end, slot, next, nslots;
  bool whole;
};
__host__ __device__ __forceinline__ Piece sk_piece(const AttnParams& p, int c, int ctas, int g,
                                                   int g1) {
  Piece pc;
  pc.head = g / p.sk_tiles_head;
  int r = g - pc.head * p.sk_tiles_head;
  int q = 0, tu = unit_tiles(p, 0);
  while (r >= tu) {
    r -= tu;
    ++q;
    tu = unit_tiles(p, q);
  }
  const int ub = g - r;
  pc.q = q;
  pc.t_begin = r;
  pc.t_end = tu < g1 - ub ? tu : g1 - ub;
  pc.slot = c - sk_owner(p, ub, ctas);
  pc.whole = pc.t_begin == 0 && pc.t_end == tu;
  pc.next = ub + pc.t_end;
  pc.nslots = sk_owner(p, ub + tu - 1, ctas) - sk_owner(p, ub, ctas) + 1;
  return pc;
}

// ============================================================================
// Kernel: two softmax warpgroups on one tcgen05 pipeline, S/P/O in TMEM.
//
// A CTA owns one q-head, one KV split and either
//   * PAIRED (two 128-row query tiles, N > 128): WG0 owns Q tile A, WG1 owns
//     Q tile B, and every K/V tile fetched by TMA feeds BOTH (M = 256 per K/V
//     tile: half the L2->SM bytes per FLOP of one tile per CTA, which is what
//     bounds this kernel at the path's skinny shapes — see
//     profiles/r01_attn_experiments.md).  MMA order per KV tile j:
//       PV_A(j-1), S_A(j), PV_B(j-1), S_B(j)   (S of one group runs while the
//     other group does its softmax);
//   * SPLIT (a single query tile, N <= 128 or an odd last tile): both groups
//     share Q and take alternate KV tiles (WG0 even, WG1 odd), MMA order
//     S_0, S_1, PV_0, S_2, PV_1, S_3 ...; the groups merge (m, l, O) at the end.
// Per group: S (128 fp32 cols) is read with tcgen05.ld, the online softmax runs
// in fp32 with exp2 (one thread per query row = TMEM lane), P is written back
// over S as packed bf16 (tcgen05.st) and consumed by the PV MMA directly from
// TMEM (A operand in tensor memory); O accumulates in TMEM across tiles and is
// rescaled in place only when a row max grows by more than 2^8.  K and V have
// separate TMA rings.  Split-KV partials go to a deterministic combine kernel.
// Warps: 0-3 WG0, 4-7 WG1, 8 TMA Q + K (+ TMEM alloc), 9 MMA, 10 TMA V.
// ============================================================================

// K/V tiles prefetched into L2 beyond the shared-memory rings (tiles ahead of
// the ring's furthest load; 0 = off).  Build-time knob; off: 2 / 4 / 8 tiles
// ahead measured 1-4 % slower (profiles/r02_attn_varlen.md) -- the K/V
// stream is bound by the L2 -> SM path, not by HBM latency.
#ifndef ASKV_ATTN_L2_PREFETCH
#define ASKV_ATTN_L2_PREFETCH 0
#endif
constexpr int kL2Prefetch = ASKV_ATTN_L2_PREFETCH;

// L2 policy of the K/V tile loads: 1 = evict_last (keep for the head's other
// query tiles), 2 = evict_first (streamed).  Build-time A/B knob.
#ifndef ASKV_ATTN_KV_POLICY
#define ASKV_ATTN_KV_POLICY 1
#endif
__device__ __forceinline__ uint64_t kv_policy() {
  return ASKV_ATTN_KV_POLICY == 2 ? l2_policy_evict_first() : l2_policy_evict_last();
}

template <int HD, bool kAllowPair>
struct Cfg {
  // K is consumed early (S) and V late (PV), so K gets the deeper ring when
  // two Q tiles take 64 KB of shared memory.
#ifndef ASKV_ATTN_PAIR_KSTAGES  // build-time A/B knobs of the paired instance's rings
#define ASKV_ATTN_PAIR_KSTAGES 3
#endif
#ifndef ASKV_ATTN_PAIR_VSTAGES
#define ASKV_ATTN_PAIR_VSTAGES 2
#endif
  static constexpr int kKStages = kAllowPair ? ASKV_ATTN_PAIR_KSTAGES : 3;
  static constexpr int kVStages = kAllowPair ? ASKV_ATTN_PAIR_VSTAGES : 3;
  static constexpr int kQTiles = kAllowPair ? 2 : 1;
  static constexpr int kChunks = HD / 64;
  static constexpr int kTileBytes = kBM * HD * 2;
  static constexpr int kQOff = 0;
  static constexpr int kKOff = kQOff + kQTiles * kTileBytes;
  static constexpr int kVOff = kKOff + kKStages * kTileBytes;
  static constexpr int kBarOff = kVOff + kVStages * kTileBytes;
  // q_full, k_full[SK], k_empty[SK], v_full[SV], v_empty[SV], s_full[2], p_full[2], o_full[2]
  static constexpr int kNumBars = 1 + 2 * kKStages + 2 * kVStages + 6;
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kSmemBytes = kTmemSlotOff + 16 + 1024;
  static constexpr uint32_t kTmemCols = 512;
  // TMEM columns: S of group w at 128*w, O of group w at 256 + 128*w
  __host__ __device__ static constexpr uint32_t col_s(int w) { return 128u * (uint32_t)w; }
  __host__ __device__ static constexpr uint32_t col_o(int w) { return 256u + 128u * (uint32_t)w; }
#ifndef ASKV_ATTN_SOFTMAX_REGS
#define ASKV_ATTN_SOFTMAX_REGS 224
#endif
  // > 0: a 12th (idle) warp completes warpgroup 2 so the producer / MMA
  // warps (56 registers each) hand their registers to the softmax
  // warpgroups (setmaxnreg).  The launch-bound cap for 11-12 warps is 168
  // registers, which spilled in the softmax (96 B/thread); with 224: no
  // spills, paired shapes -12 %, C3 -1 % (tools/kbench.py --batch 50)
#ifndef ASKV_ATTN_COLSPLIT
#define ASKV_ATTN_COLSPLIT 0
#endif
  // Column-split softmax (paired instance, d = 128): each group's 128 x 128
  // S tile is handled by two warpgroups, one per 64-column half (a thread =
  // one TMEM lane x 64 columns).  The halves share the running row max, so
  // they agree once per tile on whether a row needs the exact max (an OR
  // barrier over the two warps of the same lanes) and keep partial row sums
  // merged in the epilogue.  Halves the per-tile softmax latency that the
  // two groups' S -> softmax -> PV chains are paced by.
  static constexpr bool kCol = kAllowPair && HD == 128 && ASKV_ATTN_COLSPLIT;
  static constexpr int kSmWarps = kCol ? 16 : 8;  // softmax warps; control warps follow
  static constexpr int kCtl = kSmWarps;           // TMA Q + K, then MMA, TMA V, idle
  static constexpr int kNC = kCol ? kBN / 2 : kBN;  // S columns per softmax thread
#ifndef ASKV_ATTN_COL_REGS  // column split: softmax / control registers (sum <= 4 x 96)
#define ASKV_ATTN_COL_REGS 112
#endif
  static constexpr int kSoftmaxRegs = kCol ? ASKV_ATTN_COL_REGS : ASKV_ATTN_SOFTMAX_REGS;
  static constexpr int kCtlRegs = kCol ? 96 - 4 * (ASKV_ATTN_COL_REGS - 96) : 56;
  static constexpr int kThreads = kCol ? 640 : (kSoftmaxRegs > 0 ? 384 : 352);
#ifndef ASKV_ATTN_WARP_ARRIVE  // P-ready barrier: one arrival per softmax warp (1) or per thread (0)
#define ASKV_ATTN_WARP_ARRIVE 0
#endif
  static constexpr bool kWarpArrive = ASKV_ATTN_WARP_ARRIVE;
#ifndef ASKV_ATTN_LAST_OFULL  // o_full committed by a group's last PV only (1) or by every PV (0)
#define ASKV_ATTN_LAST_OFULL 1
#endif
#ifndef ASKV_ATTN_LAST_OFULL_ALL  // also in the unpaired instance (A/B knob)
#define ASKV_ATTN_LAST_OFULL_ALL 0
#endif
  static constexpr bool kElectIssue = ASKV_ATTN_ELECT_ISSUE;
  static constexpr bool kLastOFull = (kAllowPair || ASKV_ATTN_LAST_OFULL_ALL) && ASKV_ATTN_LAST_OFULL;  // (the unpaired instance spills with it)
  static constexpr float kRescaleLog2 = 8.0f;
  static constexpr float kRescaleLin = 256.0f;  // 2^kRescaleLog2
  static constexpr int kPolyMask = ASKV_ATTN_POLY_MASK;
  static_assert(kSmemBytes <= 232448, "smem budget");
};

template <int HD, bool kAllowPair>
__global__ void __launch_bounds__(Cfg<HD, kAllowPair>::kThreads, 1)
    attn_fwd_kernel(const __grid_constant__ CUtensorMap tm_q,
                    const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_vs, const AttnParams p,
                    const __grid_constant__ VarJobs vj) {
  using C = Cfg<HD, kAllowPair>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sK = smem + C::kKOff;
  uint8_t* sV = smem + C::kVOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + C::kKStages;
  uint64_t* v_full = k_empty + C::kKStages;
  uint64_t* v_empty = v_full + C::kVStages;
  uint64_t* s_full = v_empty + C::kVStages;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kTmemSlotOff);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // this CTA's job: the launch's only one, or (varlen) the batch job owning
  // blockIdx.x, with its rows' offsets in the shared Q / KV buffers
  int bx = blockIdx.x, h = blockIdx.y, split = blockIdx.z;
  int n_new = p.n_new, n_cached = p.n_cached, q_row0 = 0, kv_row0 = 0;
  __nv_bfloat16* out_base = p.out;
  int v_src_tiles = p.v_src_tiles;
  const int64_t* v_blk_off = p.v_blk_off;
  int64_t v_layer_row = p.v_layer_row;
  if (vj.n > 0) {
    int jb = 0;
    while (jb + 1 < vj.n && vj.j[jb + 1].cta0 <= (int)blockIdx.x) ++jb;
    const VarJob& J = vj.j[jb];
    const int local = blockIdx.x - J.cta0;
    bx = local % J.q_groups;
    h = local / J.q_groups;
    split = 0;
    n_new = J.n_new;
    n_cached = J.n_cached;
    q_row0 = J.q_row0;
    kv_row0 = J.kv_row0;
    out_base = J.out;
    v_src_tiles = J.v_src_tiles;
    v_blk_off = J.v_blk_off;
    v_layer_row = J.v_layer_row;
  }
  const int pack = p.pack;
  const int kh = pack > 1 ? h : h / p.group;
  if (threadIdx.x == 0) ATTN_TRACE(0);
  launch_stamp_begin(p.stamp);
  // Query rows of this CTA's row space: tokens of q-head h, or -- GQA packing --
  // the (token, q-head) pairs of kv head h, row = token * pack + head-in-group,
  // so one K/V tile serves 128 rows of every q-head sharing it.
  const int q_rows = pack > 1 ? n_new * pack : n_new;
  auto tok = [&](int row) { return pack > 1 ? row / pack : row; };
  auto out_row = [&](int row) -> int64_t {  // (token, q-head) index into [n_new][hq]
    return pack > 1 ? (int64_t)(row / pack) * p.hq + h * pack + row % pack
                    : (int64_t)row * p.hq + h;
  };
  // query tiles of this CTA: A at q0, B at q0 + 128 (paired only)
  const int q0 = bx * kBM * C::kQTiles;
  const int rows_a = min(kBM, q_rows - q0);
  const int rows_b = kAllowPair ? max(0, min(kBM, q_rows - q0 - kBM)) : 0;
  // CTA-uniform mode: paired when this CTA really has two query tiles
  const bool paired = rows_b > 0;
  const int last_row = q0 + (rows_b > 0 ? kBM + rows_b : rows_a) - 1;
  const int kv_end = n_cached + tok(last_row) + 1;
  const int tiles_total = (kv_end + kBN - 1) / kBN;
  const int t_begin = split * p.tiles_per_split;
  const int t_end = min(tiles_total, t_begin + p.tiles_per_split);
  const int n_tiles = t_end > t_begin ? t_end - t_begin : 0;
  const bool partial = p.num_splits > 1;
  // tiles (within the split) each paired group needs: A's last visible key is
  // n_cached + q0 + rows_a - 1, so A uses a prefix of the split's tiles
  int nt_a = n_tiles, nt_b = 0;
  if (paired) {
    const int last_a = (n_cached + tok(q0 + rows_a - 1)) / kBN;
    nt_a = max(0, min(n_tiles, last_a + 1 - t_begin));
    nt_b = rows_b > 0 ? n_tiles : 0;
  }

  if (n_tiles == 0) {  // empty split: neutral partials (CTA-uniform branch)
    if (warp < C::kSmWarps) {
      const int r = threadIdx.x & 127;
      const int g = warp / (C::kSmWarps / 2);
      const bool writer = !C::kCol || ((warp >> 2) & 1) == 0;  // one half of a row writes
      const int rows = g ? rows_b : rows_a;
      if (writer && (paired || g == 0) && r < rows) {
        const int64_t row = (int64_t)split * n_new * p.hq + out_row(q0 + g * kBM + r);
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
    for (int s = 0; s < C::kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], (C::kCol ? 2 : 1) * (C::kWarpArrive ? 4 : 128));
      mbar_init(&o_full[w], 1);
    }
    fence_mbar_init();
  }
  if (warp == C::kCtl) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) ATTN_TRACE(1);
  // kSoftmaxRegs > 0: each role branch resizes its registers first
  // (4 x 32 x kCtlRegs + kSmWarps x 32 x kSoftmaxRegs <= 64 K)
  auto shrink = [] {
    if constexpr (C::kSoftmaxRegs > 0) setmaxnreg_dec<C::kCtlRegs>();
  };

  if (warp == C::kCtl) {
    // ------------------------------------------------------------ TMA producer
    shrink();
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_vs);
      // K/V tiles are re-read by every query tile of the head: keep them in L2
      // against streaming traffic (the pre-loader's DMA writes); Q is read once.
      const uint64_t pol_kv = kv_policy();
      const uint64_t pol_q = l2_policy_evict_first();
      const int qt = paired ? 2 : 1;
      mbar_expect_tx(q_full, qt * C::kTileBytes);
      for (int t = 0; t < qt; ++t)
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d_hint(sQ + t * C::kTileBytes + c * (kBM * 128), &tm_q, q_full, c * 64,
                           pack > 1 ? h * pack : h, q_row0 + tok(q0 + t * kBM), pol_q);
      // K tiles: as far ahead as the K ring allows (S(j) needs K(j) well before
      // PV(j) needs V(j)); V tiles come from warp 10, so a V slot still held by
      // a PV in flight never delays the next K (in-kernel trace: with one
      // ordered producer the MMA warp waited ~0.55 us per tile for K(j+2)).
      for (int jk = 0; jk < n_tiles; ++jk) {
        const int st = jk % C::kKStages;
        if constexpr (kL2Prefetch > 0) {
          // pull K tiles further ahead into L2 than the shared-memory ring
          // reaches: the ring's own loads then hit L2 instead of HBM
          const int jp = jk + C::kKStages + kL2Prefetch - 1;
          if (jk == 0)
            for (int q = C::kKStages; q < jp && q < n_tiles; ++q)
#pragma unroll
              for (int c = 0; c < C::kChunks; ++c)
                tma_prefetch_l2_3d(&tm_k, c * 64, kh, kv_row0 + (t_begin + q) * kBN);
          if (jp < n_tiles)
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              tma_prefetch_l2_3d(&tm_k, c * 64, kh, kv_row0 + (t_begin + jp) * kBN);
        }
        if (jk >= C::kKStages) mbar_wait(&k_empty[st], ((jk / C::kKStages) - 1) & 1);
#if ASKV_ATTN_PROBE >= 3
        if (jk >= C::kKStages) {  // probe: no K loads after the ring's first fill
          mbar_expect_tx(&k_full[st], 0);
          continue;
        }
#endif
        mbar_expect_tx(&k_full[st], C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d_hint(sK + st * C::kTileBytes + c * (kBN * 128), &tm_k, &k_full[st],
                           c * 64, kh, kv_row0 + (t_begin + jk) * kBN, pol_kv);
      }
    }
  } else if (warp == C::kCtl + 2) {
    // ------------------------------------------------------------ TMA producer (V)
    shrink();
    if (lane == 0) {
      const uint64_t pol_kv = kv_policy();
      auto v_row = [&](int tv, bool vs) {
        return !vs ? kv_row0 + tv * kBN
               : v_blk_off ? (int)(v_blk_off[tv] / p.v_row_elems + v_layer_row)
                           : (int)(p.v_src_row0 + (int64_t)tv * kBN);
      };
      for (int jv = 0; jv < n_tiles; ++jv) {
        const int st = jv % C::kVStages;
        if constexpr (kL2Prefetch > 0) {
          const int jp = jv + C::kVStages + kL2Prefetch - 1;
          for (int q = jv == 0 ? C::kVStages : jp; q <= jp && q < n_tiles; ++q) {
            const int tq = t_begin + q;
            const bool vsq = tq < v_src_tiles;
#pragma unroll
            for (int c = 0; c < C::kChunks; ++c)
              tma_prefetch_l2_3d(vsq ? &tm_vs : &tm_v, c * 64, kh, v_row(tq, vsq));
          }
        }
        if (jv >= C::kVStages) mbar_wait(&v_empty[st], ((jv / C::kVStages) - 1) & 1);
#if ASKV_ATTN_PROBE >= 3
        if (jv >= C::kVStages) {  // probe: no V loads after the ring's first fill
          mbar_expect_tx(&v_full[st], 0);
          continue;
        }
#endif
        mbar_expect_tx(&v_full[st], C::kTileBytes);
        const int tv = t_begin + jv;
        const bool vs = tv < v_src_tiles;
        const int vrow = v_row(tv, vs);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d_hint(sV + st * C::kTileBytes + c * (kBN * 128), vs ? &tm_vs : &tm_v,
                           &v_full[st], c * 64, kh, vrow, pol_kv);
      }
    }
  } else if (warp == C::kCtl + 1) {
    // ------------------------------------------------------------ MMA issuer
    shrink();
    // kElectIssue: the whole warp runs the issue loop and each MMA / commit
    // elects its issuing lane inside the asm (no per-instruction ELECT loop)
    auto mma_ss = [](uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
      if constexpr (C::kElectIssue) umma_bf16_el(d, a, b, id, acc);
      else umma_bf16(d, a, b, id, acc);
    };
    auto mma_ts = [](uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
      if constexpr (C::kElectIssue) umma_bf16_tmem_a_el(d, a, b, id, acc);
      else umma_bf16_tmem_a(d, a, b, id, acc);
    };
    auto mma_commit = [](uint64_t* bar) {
      if constexpr (C::kElectIssue) umma_commit_el(bar);
      else umma_commit(bar);
    };
    if (C::kElectIssue || lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kBM, kBN, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kBM, HD, 0, 1);
      const uint32_t sk = smem_u32(sK), sv = smem_u32(sV);
      mbar_wait(q_full, 0);
      ATTN_TRACE(2);
      // Descriptors = base descriptor + (byte offset >> 4) in the start
      // address field (every operand lies below 256 KB of shared memory), so
      // the issuer keeps three bases live instead of a hoisted descriptor per
      // (tile, k) -- the column-split instance gives this warp 32 registers.
      const uint64_t dq = sdesc_sw128(smem_u32(sQ), 16, 1024);
      const uint64_t dk = sdesc_sw128(sk, 16, 1024);
      const uint64_t dv = sdesc_sw128(sv, kBN * 128, 1024);
      // S_w(j) = Q_w K_j^T into group w's S columns
      auto issue_s = [&](int w, int j) {
        const uint32_t qo = (paired ? w * C::kTileBytes : 0) >> 4;
        const uint32_t ko = ((j % C::kKStages) * C::kTileBytes) >> 4;
        uint64_t bq = dq + qo, bk = dk + ko;
        asm volatile("" : "+l"(bq), "+l"(bk));  // per-k sums stay immediates, not hoisted
#pragma unroll
        for (int k = 0; k < HD / 16; ++k) {
          const uint32_t off = ((k >> 2) * (kBM * 128) + (k & 3) * 32) >> 4;
          mma_ss(tmem + C::col_s(w), bq + off, bk + off, idesc_s, k > 0);
        }
        mma_commit(&s_full[w]);
      };
      // O_w += P_w V_j, P read from group w's S columns in TMEM (column
      // split: keys 0-63 at columns 0-31, keys 64-127 at 64-95 -- each half
      // writes its P over its own S columns)
      // kLastOFull: only a group's last PV signals o_full (the epilogue's
      // wait); an earlier PV's completion is implied by the s_full commit of
      // the S issued after it, which is what the softmax waits for anyway
      auto issue_pv = [&](int w, int j, bool first, bool last) {
        const uint32_t vo = ((j % C::kVStages) * C::kTileBytes) >> 4;
        uint64_t bv = dv + vo;
        uint32_t ta = tmem + C::col_s(w);
        asm volatile("" : "+l"(bv), "+r"(ta));
#pragma unroll
        for (int k = 0; k < kBN / 16; ++k)
          mma_ts(tmem + C::col_o(w),
                           ta + (C::kCol ? 64 * (k >> 2) + (k & 3) * 8 : k * 8),
                           bv + k * (16 * 128 / 16), idesc_o,
                           (!first) || (k > 0));
        if (!C::kLastOFull || last) mma_commit(&o_full[w]);
      };
      auto wait_k = [&](int j) {
#if ASKV_ATTN_PROBE == 4  // probe: no ring waits after the first fill
        if (j >= C::kKStages) return;
#endif
        mbar_wait(&k_full[j % C::kKStages], (j / C::kKStages) & 1);
        tc_fence_after();
      };
      auto wait_v = [&](int j) {
#if ASKV_ATTN_PROBE == 4
        if (j >= C::kVStages) return;
#endif
        mbar_wait(&v_full[j % C::kVStages], (j / C::kVStages) & 1);
        tc_fence_after();
      };
      if (paired) {
        wait_k(0);
        if (nt_a > 0) issue_s(0, 0);
        if (nt_b > 0) issue_s(1, 0);
        mma_commit(&k_empty[0]);
        for (int j = 0; j < n_tiles; ++j) {
          wait_v(j);
          const bool k_next = j + 1 < n_tiles;
          if (k_next) wait_k(j + 1);
#if ASKV_ATTN_INTERLEAVE
          if (HD == kBN && j + 1 < nt_a) {  // (nt_a <= nt_b: B has PV(j) and S(j+1) too)
            // PV_A(j), then S_A(j+1) k-steps interleaved with PV_B(j)'s: an
            // S MMA reads 8 KB of shared memory, a PV 4 KB, so alternating
            // them spreads the tensor core's shared-memory operand reads
            mbar_wait(&p_full[0], j & 1);
            tc_fence_after();
            issue_pv(0, j, j == 0, false);
            mbar_wait(&p_full[1], j & 1);
            tc_fence_after();
            uint64_t bq = dq, bk = dk + (((j + 1) % C::kKStages) * C::kTileBytes >> 4);
            uint64_t bv = dv + ((j % C::kVStages) * C::kTileBytes >> 4);
            uint32_t ta = tmem + C::col_s(1);
            asm volatile("" : "+l"(bq), "+l"(bk), "+l"(bv), "+r"(ta));
#pragma unroll
            for (int k = 0; k < HD / 16; ++k) {
              const uint32_t off = ((k >> 2) * (kBM * 128) + (k & 3) * 32) >> 4;
              mma_ss(tmem + C::col_s(0), bq + off, bk + off, idesc_s, k > 0);
              if (k == HD / 16 - 1) mma_commit(&s_full[0]);
              mma_ts(tmem + C::col_o(1), ta + k * 8, bv + k * (16 * 128 / 16), idesc_o,
                               j > 0 || k > 0);
            }
            if (!C::kLastOFull) mma_commit(&o_full[1]);
            mma_commit(&v_empty[j % C::kVStages]);
            if (j + 1 < nt_b) issue_s(1, j + 1);
            if (k_next) mma_commit(&k_empty[(j + 1) % C::kKStages]);
            continue;
          }
#endif
          if (j < nt_a) {
            mbar_wait(&p_full[0], j & 1);
            if (j < 28) ATTN_TRACE(64 + j);
            tc_fence_after();
            issue_pv(0, j, j == 0, j + 1 == nt_a);
            if (j + 1 < nt_a) issue_s(0, j + 1);
          }
          if (j < nt_b) {
            mbar_wait(&p_full[1], j & 1);
            if (j < 28) ATTN_TRACE(96 + j);
            tc_fence_after();
            issue_pv(1, j, j == 0, j + 1 == nt_b);
#if ASKV_ATTN_EARLY_VFREE
            // V(j)'s slot is free once PV_B(j) -- the last MMA reading it --
            // completes: commit before S_B(j+1) so the V producer does not
            // also wait for that S (B covers every tile of a paired CTA)
            mma_commit(&v_empty[j % C::kVStages]);
#endif
            if (j + 1 < nt_b) issue_s(1, j + 1);
            if (j < 28) ATTN_TRACE(160 + j);
          }
#if !ASKV_ATTN_EARLY_VFREE
          mma_commit(&v_empty[j % C::kVStages]);
#endif
          if (k_next) mma_commit(&k_empty[(j + 1) % C::kKStages]);
        }
      } else {
        wait_k(0);
        issue_s(0, 0);
        mma_commit(&k_empty[0]);
        if (n_tiles > 1) {
          wait_k(1);
          issue_s(1, 1);
          mma_commit(&k_empty[1]);
        }
        for (int j = 0; j < n_tiles; ++j) {
          const int w = j & 1;
          mbar_wait(&p_full[w], (j >> 1) & 1);
          if (j < 28) ATTN_TRACE(64 + j);
          wait_v(j);
          if (j < 28) ATTN_TRACE(96 + j);
          issue_pv(w, j, j < 2, j + 2 >= n_tiles);
          mma_commit(&v_empty[j % C::kVStages]);
          if (j < 28) ATTN_TRACE(160 + j);
          if (j + 2 < n_tiles) {
            wait_k(j + 2);
            if (j < 28) ATTN_TRACE(128 + j);
            issue_s(w, j + 2);
            mma_commit(&k_empty[(j + 2) % C::kKStages]);
          }
        }
      }
    }
  } else if (warp < C::kSmWarps) {
    // ------------------------------------------------------------ softmax groups
    if constexpr (C::kSoftmaxRegs > 0) setmaxnreg_inc<C::kSoftmaxRegs>();
    const int w = warp / (C::kSmWarps / 2);
    const int hh = C::kCol ? (warp >> 2) & 1 : 0;  // column half (column split)
    const int r = (warp & 3) * 32 + lane;  // row in tile == TMEM lane
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    // this thread's kNC S columns (P over the first kNC / 2 of them) and O half
    const uint32_t t_s = tmem + lane_off + C::col_s(w) + hh * C::kNC;
    const uint32_t t_o = tmem + lane_off + C::col_o(w);
    const uint32_t t_oh = t_o + (C::kCol ? hh * (HD / 2) : 0);
    // column split: the two warps holding the same TMEM lanes of a group
    const uint32_t pair_bar = 1 + w * 4 + (warp & 3);
    // does any row of this warp (or, column split, of its lane pair) see `v`
    auto pair_any = [&](bool v) -> bool {
      if constexpr (C::kCol) return named_bar_or(pair_bar, 64, v);
      else return __any_sync(0xffffffffu, v);
    };
    // the row max over both halves (through a free S column of each half:
    // columns kNC / 2.. are not P and S is not rewritten before p_full)
    auto pair_max = [&](float m) -> float {
      if constexpr (C::kCol) {
        tmem_st2(t_s + C::kNC / 2, m, m);
        tmem_wait_st();
        tc_fence_before();
        named_bar_sync(pair_bar, 64);
        tc_fence_after();
        float a, b;
        tmem_ld2(tmem + lane_off + C::col_s(w) + (hh ^ 1) * C::kNC + C::kNC / 2, a, b);
        return fmaxf(m, a);
      } else {
        return m;
      }
    };
    const int qt0 = q0 + (paired ? w * kBM : 0);  // first query of this group's tile
    const int row_limit = n_cached + tok(qt0 + r);
    const float sl2 = p.scale_log2;
    const int my_tiles = paired ? (w ? nt_b : nt_a) : (n_tiles - w + 1) / 2;
    float m_acc = -INFINITY, l_acc = 0.f;
    // One tile of the online softmax.  The whole 128-column S row is pulled
    // into registers with four back-to-back tcgen05.ld and a single wait, so
    // the max pass and the exp pass read registers, not TMEM; the column mask
    // exists only in the diagonal-tile instance (kMask), keeping the common
    // off-diagonal tile free of per-element selects.
    auto tile = [&](auto mask_tag, int t, int lim) {
      constexpr bool kMask = decltype(mask_tag)::value;
      uint32_t sr[C::kNC];
#if ASKV_ATTN_PROBE > 0
      // Pipeline probes (tools/attn_varlen_trace.cu only; the output is not
      // attention): 1 = no softmax work at all, 2 = the S loads only, 3 = as
      // 1 and no K/V loads after the rings' first fill (the producers arrive
      // on the full barriers without a copy), 4 = as 3 and the MMA warp does
      // not wait on the ring barriers after the first fill.  They time the MMA / TMA
      // pipeline of the real kernel without the softmax.
      if (ASKV_ATTN_PROBE == 2) {
#pragma unroll
        for (int c = 0; c < C::kNC / 32; ++c)
          tmem_ld32_nowait(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
        tmem_wait_ld();
        uint32_t x = 0;
#pragma unroll
        for (int e = 0; e < C::kNC; ++e) x ^= sr[e];
        if (x == 0x7fc00001u) l_acc += 1.f;  // keep the loads
      }
      tc_fence_before();
      __syncwarp();
      if (!C::kWarpArrive || elect_one()) mbar_arrive(&p_full[w]);
      return;
#endif
#pragma unroll
      for (int c = 0; c < C::kNC / 32; ++c)
        tmem_ld32_nowait(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
      tmem_wait_ld();
      const bool trace_t = threadIdx.x == 0 && t >= 2 && t < 18;
      if (trace_t) ATTN_TRACE(192 + 4 * (t - 2));
      const float2 sl2v = make_float2(sl2, sl2);
      float2 ls0 = make_float2(0.f, 0.f), ls1 = ls0, ls2 = ls0, ls3 = ls0;
      // exps of the row against -neg_m, P (bf16 pairs) over the S columns
      // already read, row sums into ls*; kTrack: max of the raw scores of the
      // polynomial lanes into *pmax.  Pair slot (e / 2) % 8 of each 16 goes to
      // the FMA pipe (packed cubic) when bit slot of kPolyMask is set, so MUFU
      // and FMA share the load; masked tiles keep MUFU (exact zeros).
      auto exps = [&](auto track_tag, float neg_m, float* pmax) {
        constexpr bool kTrack = decltype(track_tag)::value;
        const float2 negm2 = make_float2(neg_m, neg_m);
        ls0 = ls1 = ls2 = ls3 = make_float2(0.f, 0.f);
        float pm = -INFINITY;
#pragma unroll
        for (int c = 0; c < C::kNC / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int k = c * 32 + e;
            const float2 x = ffma2(
                make_float2(__uint_as_float(sr[k]), __uint_as_float(sr[k + 1])), sl2v, negm2);
            const bool poly = !kMask && ((C::kPolyMask >> ((e >> 1) & 7)) & 1);
            if (kTrack && poly) pm = fmax3(pm, __uint_as_float(sr[k]), __uint_as_float(sr[k + 1]));
            const float2 pp = poly ? ex2_poly2(x) : make_float2(ex2(x.x), ex2(x.y));
            switch ((e >> 1) & 3) {
              case 0: ls0 = fadd2(ls0, pp); break;
              case 1: ls1 = fadd2(ls1, pp); break;
              case 2: ls2 = fadd2(ls2, pp); break;
              default: ls3 = fadd2(ls3, pp); break;
            }
            pk[e >> 1] = pack_bf16x2(pp.x, pp.y);
          }
          tmem_st16(t_s + c * 16, pk);
        }
        if (kTrack) *pmax = pm;
      };
      // O_w holds this group's tiles < t (their last PV complete): rescale it
      // in place by 2^(m_acc - m_tile) where a row's max grew past the threshold
      auto rescale = [&](float m_tile, bool need) {
        tc_fence_after();
        const float f = need ? ex2(m_acc - m_tile) : 1.f;
#pragma unroll 1
        for (int c = 0; c < (C::kCol ? HD / 2 : HD) / 32; ++c) {
          float ov[32];
          tmem_ld32(t_oh + c * 32, ov);
#pragma unroll
          for (int e = 0; e < 32; ++e) ov[e] *= f;
          tmem_st32(t_oh + c * 32, ov);
        }
        tmem_wait_st();
        if (need) {
          l_acc *= f;
          m_acc = m_tile;
        }
      };
      auto row_max = [&]() {
        float a0 = fmaxf(__uint_as_float(sr[0]), __uint_as_float(sr[1]));
        float a1 = fmaxf(__uint_as_float(sr[2]), __uint_as_float(sr[3]));
        float a2 = fmaxf(__uint_as_float(sr[4]), __uint_as_float(sr[5]));
        float a3 = fmaxf(__uint_as_float(sr[6]), __uint_as_float(sr[7]));
#pragma unroll
        for (int e = 8; e < C::kNC; e += 8) {
          a0 = fmax3(a0, __uint_as_float(sr[e + 0]), __uint_as_float(sr[e + 1]));
          a1 = fmax3(a1, __uint_as_float(sr[e + 2]), __uint_as_float(sr[e + 3]));
          a2 = fmax3(a2, __uint_as_float(sr[e + 4]), __uint_as_float(sr[e + 5]));
          a3 = fmax3(a3, __uint_as_float(sr[e + 6]), __uint_as_float(sr[e + 7]));
        }
        return fmax3(fmax3(a0, a1, a2), a3, -INFINITY) * sl2;
      };
      // Every o_full phase is consumed (compute-sanitizer synccheck flags a
      // phase nobody waits for): with kLastOFull there is one per group, the
      // epilogue's; otherwise every PV commits one and it is waited here.
      // Free either way: s_full of S(t) was committed after PV(t-1) was
      // issued, and a commit tracks every earlier tcgen05 op of the issuing
      // thread, so PV(t-1) is already complete.
      auto consume_pv = [&] {
        if (!C::kLastOFull && t > 0) mbar_wait(&o_full[w], (t - 1) & 1);
      };
      bool done = false;
#if ASKV_ATTN_SUMCHECK
      if (!kMask && t > 0 && __all_sync(0xffffffffu, m_acc > -INFINITY)) {
        // No max pass: exps straight against m_acc.  A row needs the lazy
        // rescale only if some exponent exceeds 2^kRescaleLog2; its MUFU lanes
        // then push the row sum past 2^kRescaleLog2 (inf included) and its
        // polynomial lanes are checked through their raw max.  Only then is
        // the exact max taken and, if it crossed the threshold, the row
        // rescaled and the tile redone -- the values the max-first order gives.
        float pmax;
        exps(std::true_type{}, -m_acc, &pmax);
        const float2 la = fadd2(ls0, ls1), lb = fadd2(ls2, ls3);
        const float lsum = (la.x + la.y) + (lb.x + lb.y);
        const bool over = !(lsum <= C::kRescaleLin) ||
                          pmax * sl2 > m_acc + C::kRescaleLog2;
        if (trace_t) ATTN_TRACE(193 + 4 * (t - 2));
        consume_pv();
        if (pair_any(over)) {
          const float m_tile = pair_max(row_max());
          const bool need = m_tile > m_acc + C::kRescaleLog2;
          if (__any_sync(0xffffffffu, need)) {
            tmem_wait_st();  // the first pass's P stores land before the redo's
            rescale(m_tile, need);
            exps(std::false_type{}, -m_acc, nullptr);
          }
        }
        done = true;
      }
#endif
      if (!done) {
        if (kMask) {
#pragma unroll
          for (int e = 0; e < C::kNC; ++e) sr[e] = (e <= lim) ? sr[e] : 0xff800000u;  // -inf
        }
        const float m_tile = pair_max(row_max());
        const bool need = m_tile > m_acc + C::kRescaleLog2;
        if (trace_t) ATTN_TRACE(193 + 4 * (t - 2));
        consume_pv();
        if (t == 0) {
          if (need) m_acc = m_tile;
        } else if (__any_sync(0xffffffffu, need)) {
          rescale(m_tile, need);
        }
        exps(std::false_type{}, (m_acc == -INFINITY) ? 0.f : -m_acc, nullptr);
      }
      const float2 la = fadd2(ls0, ls1), lb = fadd2(ls2, ls3);
      l_acc += (la.x + la.y) + (lb.x + lb.y);
      if (trace_t) ATTN_TRACE(194 + 4 * (t - 2));
      tmem_wait_st();
      tc_fence_before();
      if constexpr (C::kWarpArrive) {
        // one arrival per warp: the warp-collective wait::st above completed
        // every lane's P stores; 4 instead of 128 arrivals on the barrier the
        // MMA warp waits on
        __syncwarp();
        if (elect_one()) mbar_arrive(&p_full[w]);
      } else {
        mbar_arrive(&p_full[w]);
      }
    };
    for (int t = 0; t < my_tiles; ++t) {
      const int j = paired ? t : 2 * t + w;
      mbar_wait(&s_full[w], t & 1);
      if (threadIdx.x == 0 && t < 28) ATTN_TRACE(8 + 2 * t);
      tc_fence_after();
      const int kbase = (t_begin + j) * kBN;
      // group-uniform: does any row of this tile see a masked column here?
      if (kbase + kBN - 1 > n_cached + tok(qt0))
        tile(std::true_type{}, t, row_limit - kbase - hh * C::kNC);
      else
        tile(std::false_type{}, t, 0);
      if (threadIdx.x == 0 && t < 28) ATTN_TRACE(9 + 2 * t);
      // P-done of WG0's other warps (per-warp skew of the p_full arrival)
      if (lane == 0 && w == 0 && (warp & 3) != 0 && t < 4) ATTN_TRACE(180 + 3 * t + (warp & 3) - 1);
    }
    if (my_tiles > 0) {  // this group's last PV
      mbar_wait(&o_full[w], C::kLastOFull ? 0 : (my_tiles - 1) & 1);
      tc_fence_after();
    }
    if (threadIdx.x == 0) ATTN_TRACE(3);
    // ---- epilogue
    float m_fin = m_acc, l_fin = l_acc, f_self = l_acc > 0.f ? 1.f : 0.f, f_other = 0.f;
    int col0 = 0, ncols = HD;
    if constexpr (C::kCol) {
      // (m, partial l) of each half through a free S column (S / P are dead
      // after the last PV); unpaired, the groups' (m, l) merge as below and a
      // thread writes a quarter of the columns
      tmem_st2(t_s + C::kNC / 2, m_acc, l_acc);
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(9, 32 * C::kSmWarps);
      tc_fence_after();
      float mg[2], lg[2];
      for (int g = 0; g < (paired ? 1 : 2); ++g) {
        const int gg = paired ? w : g;
        float m0, l0, m1, l1;
        tmem_ld2(tmem + lane_off + C::col_s(gg) + C::kNC / 2, m0, l0);
        tmem_ld2(tmem + lane_off + C::col_s(gg) + C::kNC + C::kNC / 2, m1, l1);
        mg[g] = m0;
        lg[g] = l0 + l1;
      }
      if (paired) {
        l_fin = lg[0];
        f_self = l_fin > 0.f ? 1.f : 0.f;
        col0 = hh * (HD / 2);
        ncols = HD / 2;
      } else {
        m_fin = fmaxf(mg[0], mg[1]);
        const float f0 = lg[0] > 0.f ? ex2(mg[0] - m_fin) : 0.f;
        const float f1 = lg[1] > 0.f ? ex2(mg[1] - m_fin) : 0.f;
        l_fin = lg[0] * f0 + lg[1] * f1;
        f_self = w ? f1 : f0;
        f_other = w ? f0 : f1;
        col0 = (w * 2 + hh) * (HD / 4);
        ncols = HD / 4;
      }
    } else if (!paired) {
      // merge the two groups' (m, l, O) through TMEM; each writes half the columns
      tmem_st2(t_s + 64, m_acc, l_acc);  // S columns are free after the last PV
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(1, 256);
      tc_fence_after();
      float m0, l0, m1, l1;
      tmem_ld2(tmem + lane_off + C::col_s(0) + 64, m0, l0);
      tmem_ld2(tmem + lane_off + C::col_s(1) + 64, m1, l1);
      m_fin = fmaxf(m0, m1);
      const float f0 = l0 > 0.f ? ex2(m0 - m_fin) : 0.f;
      const float f1 = l1 > 0.f ? ex2(m1 - m_fin) : 0.f;
      l_fin = l0 * f0 + l1 * f1;
      f_self = w ? f1 : f0;
      f_other = w ? f0 : f1;
      col0 = w * (HD / 2);
      ncols = HD / 2;
    }
    const float inv_l = l_fin > 0.f ? 1.f / l_fin : 0.f;
    const int rows_g = paired ? (w ? rows_b : rows_a) : rows_a;
    const int qi = qt0 + r;
    const uint32_t t_o_other = tmem + lane_off + C::col_o(w ^ 1);
    for (int c = 0; c < ncols / 32; ++c) {
      const int col = col0 + c * 32;
      float a[32], b[32];
      tmem_ld32(t_o + col, a);
      if (!paired) tmem_ld32(t_o_other + col, b);
      float o[32];
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float x = f_self > 0.f ? a[e] * f_self : 0.f;
        const float y = (!paired && f_other > 0.f) ? b[e] * f_other : 0.f;
        o[e] = (x + y) * inv_l;
      }
      if (r < rows_g) {
        if (!partial) {
          __nv_bfloat16* dst = out_base + out_row(qi) * HD + col;
#pragma unroll
          for (int e = 0; e < 32; e += 8) {
            uint4 v;
            v.x = pack_bf16x2(o[e + 0], o[e + 1]);
            v.y = pack_bf16x2(o[e + 2], o[e + 3]);
            v.z = pack_bf16x2(o[e + 4], o[e + 5]);
            v.w = pack_bf16x2(o[e + 6], o[e + 7]);
            *reinterpret_cast<uint4*>(dst + e) = v;
          }
        } else {
          const int64_t row = (int64_t)split * n_new * p.hq + out_row(qi);
          float4* po = reinterpret_cast<float4*>(p.part_o + row * HD + col);
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            po[e / 4] = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
          if (c == 0 && col0 == 0)
            p.part_lse[row] = l_fin > 0.f ? m_fin + __log2f(l_fin) : -INFINITY;
        }
      }
    }
  } else {
    shrink();  // warp 11: completes warpgroup 2 for setmaxnreg
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::kCtl) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
  if (threadIdx.x == 0) ATTN_TRACE(4);
  if (p.num_splits == 1) launch_stamp_end(p.stamp);
}

// ============================================================================
// Stream-K kernel (single query tile per unit, the non-paired shapes; opt-in).
//
// Units (query tile, head) are too few to fill 148 SMs at the path's skinny
// shapes (C3 p50: 2 query tiles x 40 heads = 80 CTAs) and splitting them
// uniformly costs a second wave.  Instead the KV tiles of all units form one
// head-major list cut into gridDim.x (<= #SMs) equal contiguous ranges: each
// CTA walks its range as a sequence of pieces (a piece = a run of one unit's
// KV tiles), re-loading Q at each unit boundary.  A piece covering a whole
// unit writes the bf16 output (staged in shared memory, TMA store); a unit
// cut across CTAs leaves one fp32 partial (O, lse) per piece and bumps the
// unit's arrival counter -- the piece that arrives last merges all slots in
// slot order (deterministic) and writes the output, so there is no separate
// combine pass.  Warp roles and the per-tile pipeline are the SPLIT mode of
// attn_fwd_kernel; the ring / phase counters run on across pieces, q_empty
// (MMA -> Q producer) guards the Q tile and o_free (softmax -> MMA) the
// TMEM S / O columns between pieces.
// ============================================================================
template <int HD>
struct SkCfg {
  using B = Cfg<HD, false>;
  static constexpr int kKStages = B::kKStages;
  // V is consumed last (PV): 2 stages suffice (the paired kernel runs with 2)
  // and free a 128 x HD bf16 tile that stages the output for its TMA store
  static constexpr int kVStages = 2;
  static constexpr int kChunks = B::kChunks;
  static constexpr int kTileBytes = B::kTileBytes;
  static constexpr int kQOff = B::kQOff, kKOff = B::kKOff, kVOff = B::kVOff;
  static constexpr int kStageOff = kVOff + kVStages * kTileBytes;
  static constexpr int kBarOff = kStageOff + kTileBytes;
  static constexpr int kNumBars = 1 + 2 * kKStages + 2 * kVStages + 6 + 2;  // + q_empty, o_free
  static constexpr int kTmemSlotOff = kBarOff + kNumBars * 8;
  static constexpr int kSmemBytes = kTmemSlotOff + 16 + 1024;
  static constexpr uint32_t kTmemCols = B::kTmemCols;
  static constexpr int kSoftmaxRegs = B::kSoftmaxRegs;
  static constexpr int kThreads = B::kThreads;
  static constexpr float kRescaleLog2 = B::kRescaleLog2;
  __host__ __device__ static constexpr uint32_t col_s(int w) { return B::col_s(w); }
  __host__ __device__ static constexpr uint32_t col_o(int w) { return B::col_o(w); }
  static_assert(kSmemBytes <= 232448, "smem budget");
};

template <int HD>
__global__ void __launch_bounds__(ASKV_ATTN_SOFTMAX_REGS > 0 ? 384 : 352, 1)
    attn_sk_kernel(const __grid_constant__ CUtensorMap tm_q,
                   const __grid_constant__ CUtensorMap tm_k,
                   const __grid_constant__ CUtensorMap tm_v,
                   const __grid_constant__ CUtensorMap tm_vs,
                   const __grid_constant__ CUtensorMap tm_o, const AttnParams p) {
  using C = SkCfg<HD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem + C::kQOff;
  uint8_t* sK = smem + C::kKOff;
  uint8_t* sV = smem + C::kVOff;
  uint8_t* sStage = smem + C::kStageOff;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::kBarOff);
  uint64_t* q_full = bars;
  uint64_t* k_full = q_full + 1;
  uint64_t* k_empty = k_full + C::kKStages;
  uint64_t* v_full = k_empty + C::kKStages;
  uint64_t* v_empty = v_full + C::kVStages;
  uint64_t* s_full = v_empty + C::kVStages;
  uint64_t* p_full = s_full + 2;
  uint64_t* o_full = p_full + 2;
  uint64_t* q_empty = o_full + 2;
  uint64_t* o_free = q_empty + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + C::kTmemSlotOff);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int ctas = gridDim.x;
  const int cta = blockIdx.x;
  const int pack = p.pack;
  const int q_rows = pack > 1 ? p.n_new * pack : p.n_new;
  auto tok = [&](int row) { return pack > 1 ? row / pack : row; };
  auto out_row = [&](int h, int row) -> int64_t {
    return pack > 1 ? (int64_t)(row / pack) * p.hq + h * pack + row % pack
                    : (int64_t)row * p.hq + h;
  };
  if (threadIdx.x == 0) ATTN_TRACE(0);
  launch_stamp_begin(p.stamp);
  int g0, g1;
  sk_range(p, cta, ctas, g0, g1);
  if (g0 >= g1) return;  // CTA-uniform (the host launches <= sk_total CTAs)

  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    mbar_init(o_free, 8);  // one arrival per softmax warp
    for (int s = 0; s < C::kKStages; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < C::kVStages; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    for (int w = 0; w < 2; ++w) {
      mbar_init(&s_full[w], 1);
      mbar_init(&p_full[w], 128);
      mbar_init(&o_full[w], 1);
    }
    fence_mbar_init();
  }
  if (warp == 8) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  if (threadIdx.x == 0) ATTN_TRACE(1);
  auto shrink = [] {
    if constexpr (C::kSoftmaxRegs > 0) setmaxnreg_dec<56>();
  };

  if (warp == 8) {
    // ------------------------------------------------------------ TMA: Q per piece, K tiles
    shrink();
    if (lane == 0) {
      tma_prefetch_desc(&tm_q);
      tma_prefetch_desc(&tm_k);
      tma_prefetch_desc(&tm_v);
      tma_prefetch_desc(&tm_vs);
      const uint64_t pol_kv = l2_policy_evict_last();
      const uint64_t pol_q = l2_policy_evict_first();
      int jk = 0, np = 0;
      for (int g = g0; g < g1; ++np) {
        const Piece pc = sk_piece(p, cta, ctas, g, g1);
        g = pc.next;
        const int kh = pack > 1 ? pc.head : pc.head / p.group;
        if (np > 0) mbar_wait(q_empty, (np - 1) & 1);  // every S of the previous piece done
        mbar_expect_tx(q_full, C::kTileBytes);
#pragma unroll
        for (int c = 0; c < C::kChunks; ++c)
          tma_load_3d_hint(sQ + c * (kBM * 128), &tm_q, q_full, c * 64,
                           pack > 1 ? pc.head * pack : pc.head, tok(pc.q * kBM), pol_q);
        for (int t = pc.t_begin; t < pc.t_end; ++t, ++jk) {
          const int st = jk % C::kKStages;
          if (jk >= C::kKStages) mbar_wait(&k_empty[st], ((jk / C::kKStages) - 1) & 1);
          mbar_expect_tx(&k_full[st], C::kTileBytes);
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d_hint(sK + st * C::kTileBytes + c * (kBN * 128), &tm_k, &k_full[st],
                             c * 64, kh, t * kBN, pol_kv);
        }
      }
    }
  } else if (warp == 10) {
    // ------------------------------------------------------------ TMA: V tiles
    shrink();
    if (lane == 0) {
      const uint64_t pol_kv = l2_policy_evict_last();
      int jv = 0;
      for (int g = g0; g < g1;) {
        const Piece pc = sk_piece(p, cta, ctas, g, g1);
        g = pc.next;
        const int kh = pack > 1 ? pc.head : pc.head / p.group;
        for (int t = pc.t_begin; t < pc.t_end; ++t, ++jv) {
          const int st = jv % C::kVStages;
          if (jv >= C::kVStages) mbar_wait(&v_empty[st], ((jv / C::kVStages) - 1) & 1);
          mbar_expect_tx(&v_full[st], C::kTileBytes);
          bool vs;
          const int vrow = v_tile_row(p, t, vs);
#pragma unroll
          for (int c = 0; c < C::kChunks; ++c)
            tma_load_3d_hint(sV + st * C::kTileBytes + c * (kBN * 128), vs ? &tm_vs : &tm_v,
                             &v_full[st], c * 64, kh, vrow, pol_kv);
        }
      }
    }
  } else if (warp == 9) {
    // ------------------------------------------------------------ MMA issuer
    shrink();
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(kBM, kBN, 0, 0);
      constexpr uint32_t idesc_o = idesc_bf16_f32(kBM, HD, 0, 1);
      const uint32_t sk = smem_u32(sK), sv = smem_u32(sV), sq = smem_u32(sQ);
      int jb = 0, np = 0;
      int cnt0 = 0, cnt1 = 0;  // tiles each softmax group finished in earlier pieces
      for (int g = g0; g < g1; ++np) {
        const Piece pc = sk_piece(p, cta, ctas, g, g1);
        g = pc.next;
        const bool last_piece = g >= g1;
        const int n = pc.t_end - pc.t_begin;
        mbar_wait(q_full, np & 1);
        if (np < 4) ATTN_TRACE(40 + 2 * np);
        if (np > 0) mbar_wait(o_free, (np - 1) & 1);  // S / O columns released
        if (np < 4) ATTN_TRACE(41 + 2 * np);
        tc_fence_after();
        auto issue_s = [&](int w, int j) {
          const uint32_t kb = sk + ((jb + j) % C::kKStages) * C::kTileBytes;
#pragma unroll
          for (int k = 0; k < HD / 16; ++k) {
            const uint32_t off = (k >> 2) * (kBM * 128) + (k & 3) * 32;
            umma_bf16(tmem + C::col_s(w), sdesc_sw128(sq + off, 16, 1024),
                      sdesc_sw128(kb + off, 16, 1024), idesc_s, k > 0);
          }
          umma_commit(&s_full[w]);
          // the piece's last reader of Q (the last piece's phase has no waiter)
          if (j == n - 1 && !last_piece) umma_commit(q_empty);
        };
        auto issue_pv = [&](int w, int j, bool first) {
          const uint32_t vb = sv + ((jb + j) % C::kVStages) * C::kTileBytes;
#pragma unroll
          for (int k = 0; k < kBN / 16; ++k)
            umma_bf16_tmem_a(tmem + C::col_o(w), tmem + C::col_s(w) + k * 8,
                             sdesc_sw128(vb + k * (16 * 128), kBN * 128, 1024), idesc_o,
                             (!first) || (k > 0));
          umma_commit(&o_full[w]);
        };
        auto wait_k = [&](int j) {
          mbar_wait(&k_full[(jb + j) % C::kKStages], ((jb + j) / C::kKStages) & 1);
          tc_fence_after();
        };
        auto wait_v = [&](int j) {
          mbar_wait(&v_full[(jb + j) % C::kVStages], ((jb + j) / C::kVStages) & 1);
          tc_fence_after();
        };
        wait_k(0);
        issue_s(0, 0);
        umma_commit(&k_empty[jb % C::kKStages]);
        if (n > 1) {
          wait_k(1);
          issue_s(1, 1);
          umma_commit(&k_empty[(jb + 1) % C::kKStages]);
        }
        for (int j = 0; j < n; ++j) {
          const int w = j & 1;
          mbar_wait(&p_full[w], ((w ? cnt1 : cnt0) + (j >> 1)) & 1);
          if (jb + j < 28) ATTN_TRACE(64 + jb + j);
          wait_v(j);
          if (jb + j < 28) ATTN_TRACE(96 + jb + j);
          issue_pv(w, j, j < 2);
          if (jb + j < 28) ATTN_TRACE(160 + jb + j);
          umma_commit(&v_empty[(jb + j) % C::kVStages]);
          if (j + 2 < n) {
            wait_k(j + 2);
            if (jb + j < 28) ATTN_TRACE(128 + jb + j);
            issue_s(w, j + 2);
            umma_commit(&k_empty[(jb + j + 2) % C::kKStages]);
          }
        }
        cnt0 += (n + 1) / 2;
        cnt1 += n / 2;
        jb += n;
      }
    }
  } else if (warp < 8) {
    // ------------------------------------------------------------ softmax groups
    if constexpr (C::kSoftmaxRegs > 0) setmaxnreg_inc<C::kSoftmaxRegs>();
    const int w = warp >> 2;
    const int r = (warp & 3) * 32 + lane;
    const uint32_t lane_off = (uint32_t)((warp & 3) * 32) << 16;
    const uint32_t t_s = tmem + lane_off + C::col_s(w);
    const uint32_t t_o = tmem + lane_off + C::col_o(w);
    const float sl2 = p.scale_log2;
    int cw = 0;  // this group's tiles in earlier pieces (barrier phases)
    for (int g = g0; g < g1;) {
      const Piece pc = sk_piece(p, cta, ctas, g, g1);
      g = pc.next;
      const int n = pc.t_end - pc.t_begin;
      const int my_tiles = (n - w + 1) / 2;
      const int qt0 = pc.q * kBM;
      const int row_limit = p.n_cached + tok(qt0 + r);
      float m_acc = -INFINITY, l_acc = 0.f;
      auto tile = [&](auto mask_tag, int t, int lim) {
        constexpr bool kMask = decltype(mask_tag)::value;
        uint32_t sr[kBN];
#pragma unroll
        for (int c = 0; c < kBN / 32; ++c)
          tmem_ld32_nowait(t_s + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sr[c * 32]));
        tmem_wait_ld();
        if (kMask) {
#pragma unroll
          for (int e = 0; e < kBN; ++e) sr[e] = (e <= lim) ? sr[e] : 0xff800000u;
        }
        float a0 = fmaxf(__uint_as_float(sr[0]), __uint_as_float(sr[1]));
        float a1 = fmaxf(__uint_as_float(sr[2]), __uint_as_float(sr[3]));
        float a2 = fmaxf(__uint_as_float(sr[4]), __uint_as_float(sr[5]));
        float a3 = fmaxf(__uint_as_float(sr[6]), __uint_as_float(sr[7]));
#pragma unroll
        for (int e = 8; e < kBN; e += 8) {
          a0 = fmax3(a0, __uint_as_float(sr[e + 0]), __uint_as_float(sr[e + 1]));
          a1 = fmax3(a1, __uint_as_float(sr[e + 2]), __uint_as_float(sr[e + 3]));
          a2 = fmax3(a2, __uint_as_float(sr[e + 4]), __uint_as_float(sr[e + 5]));
          a3 = fmax3(a3, __uint_as_float(sr[e + 6]), __uint_as_float(sr[e + 7]));
        }
        const float m_tile = fmax3(fmax3(a0, a1, a2), a3, -INFINITY) * sl2;
        const bool need = m_tile > m_acc + C::kRescaleLog2;
        if (t > 0) mbar_wait(&o_full[w], (cw + t - 1) & 1);  // PV(t-1) of this group
        if (t == 0) {
          if (need) m_acc = m_tile;
        } else if (__any_sync(0xffffffffu, need)) {
          tc_fence_after();
          const float f = need ? ex2(m_acc - m_tile) : 1.f;
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            float ov[32];
            tmem_ld32(t_o + c * 32, ov);
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] *= f;
            tmem_st32(t_o + c * 32, ov);
          }
          tmem_wait_st();
          if (need) {
            l_acc *= f;
            m_acc = m_tile;
          }
        }
        const float neg_m = (m_acc == -INFINITY) ? 0.f : -m_acc;
        const float2 sl2v = make_float2(sl2, sl2), negm2 = make_float2(neg_m, neg_m);
        float2 ls0 = make_float2(0.f, 0.f), ls1 = ls0, ls2 = ls0, ls3 = ls0;
#pragma unroll
        for (int c = 0; c < kBN / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 32; e += 2) {
            const int k = c * 32 + e;
            const float2 x = ffma2(make_float2(__uint_as_float(sr[k]), __uint_as_float(sr[k + 1])),
                                   sl2v, negm2);
            const float2 pp = (!kMask && ((e >> 1) & 3) >= 4 - ASKV_ATTN_POLY_Q) ? ex2_poly2(x)
                                                               : make_float2(ex2(x.x), ex2(x.y));
            switch ((e >> 1) & 3) {
              case 0: ls0 = fadd2(ls0, pp); break;
              case 1: ls1 = fadd2(ls1, pp); break;
              case 2: ls2 = fadd2(ls2, pp); break;
              default: ls3 = fadd2(ls3, pp); break;
            }
            pk[e >> 1] = pack_bf16x2(pp.x, pp.y);
          }
          tmem_st16(t_s + c * 16, pk);
        }
        const float2 la = fadd2(ls0, ls1), lb = fadd2(ls2, ls3);
        l_acc += (la.x + la.y) + (lb.x + lb.y);
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(&p_full[w]);
      };
      for (int t = 0; t < my_tiles; ++t) {
        const int j = 2 * t + w;
        mbar_wait(&s_full[w], (cw + t) & 1);
        if (threadIdx.x == 0 && cw + t < 14) ATTN_TRACE(8 + 2 * (cw + t));
        tc_fence_after();
        const int kbase = (pc.t_begin + j) * kBN;
        if (kbase + kBN - 1 > p.n_cached + tok(qt0))
          tile(std::true_type{}, t, row_limit - kbase);
        else
          tile(std::false_type{}, t, 0);
        if (threadIdx.x == 0 && cw + t < 14) ATTN_TRACE(9 + 2 * (cw + t));
      }
      if (threadIdx.x == 0) ATTN_TRACE(3);
      if (my_tiles > 0) {
        mbar_wait(&o_full[w], (cw + my_tiles - 1) & 1);
        tc_fence_after();
      }
      // ---- merge the two groups' (m, l, O) through TMEM; each takes half the columns.
      // Everything this piece needs from TMEM is pulled into registers first,
      // then o_free lets the next piece's MMAs start while the partial is
      // stored (column-major per unit, so a warp's 32 rows of one column are
      // one coalesced 128-byte store).
      tmem_st2(t_s + 64, m_acc, l_acc);
      tmem_wait_st();
      tc_fence_before();
      named_bar_sync(1, 256);
      tc_fence_after();
      float m0, l0, m1, l1;
      tmem_ld2(tmem + lane_off + C::col_s(0) + 64, m0, l0);
      tmem_ld2(tmem + lane_off + C::col_s(1) + 64, m1, l1);
      const float m_fin = fmaxf(m0, m1);
      const float f0 = l0 > 0.f ? ex2(m0 - m_fin) : 0.f;
      const float f1 = l1 > 0.f ? ex2(m1 - m_fin) : 0.f;
      const float l_fin = l0 * f0 + l1 * f1;
      const float f_self = w ? f1 : f0, f_other = w ? f0 : f1;
      const int col0 = w * (HD / 2);
      const float inv_l = l_fin > 0.f ? 1.f / l_fin : 0.f;
      const uint32_t t_o_other = tmem + lane_off + C::col_o(w ^ 1);
      constexpr int kHalf = HD / 2;
      float o[kHalf];
#pragma unroll
      for (int c = 0; c < kHalf / 32; ++c) {
        float a[32], b[32];
        tmem_ld32(t_o + col0 + c * 32, a);
        tmem_ld32(t_o_other + col0 + c * 32, b);
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float x = f_self > 0.f ? a[e] * f_self : 0.f;
          const float y = f_other > 0.f ? b[e] * f_other : 0.f;
          o[c * 32 + e] = (x + y) * inv_l;
        }
      }
      // S / O columns of both groups are read: the next piece may overwrite them
      if (g < g1) {
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(o_free);
      }
      // ---- output.  A whole unit is final; a cut unit leaves its partial
      // (column-major, coalesced) and counts its arrival: the piece that
      // arrives last merges every slot (deterministic slot order) and writes
      // the unit's output -- no separate combine pass.
      if (threadIdx.x == 0) ATTN_TRACE(176);
      const int u = pc.head * p.sk_q_tiles + pc.q;
      const float lse_own = l_fin > 0.f ? m_fin + __log2f(l_fin) : -INFINITY;
      bool final_here = pc.whole;
      if (!pc.whole) {
        const int64_t slab = (int64_t)pc.slot * p.sk_units + u;
        float* po = p.part_o + (slab * HD + col0) * kBM + r;
#pragma unroll
        for (int e = 0; e < kHalf; ++e) po[e * kBM] = o[e];
        if (w == 0) p.part_lse[slab * kBM + r] = lse_own;
        if (threadIdx.x == 0) ATTN_TRACE(177);
        __threadfence();
        named_bar_sync(2, 256);
        if (threadIdx.x == 0) ATTN_TRACE(178);
        if (threadIdx.x == 0) {
          const int old = atomicAdd(p.sk_cnt + u, 1);
          const int last = old == pc.nslots - 1;
          if (last) p.sk_cnt[u] = 0;   // every piece of the unit has counted
          tmem_slot[1] = last;
        }
        named_bar_sync(2, 256);
        final_here = tmem_slot[1] != 0;
        if (threadIdx.x == 0) ATTN_TRACE(179);
        if (final_here) {
          __threadfence();
          float mx = lse_own;
          for (int s2 = 0; s2 < pc.nslots; ++s2)
            if (s2 != pc.slot)
              mx = fmaxf(mx, p.part_lse[((int64_t)s2 * p.sk_units + u) * kBM + r]);
          const float w_own = lse_own == -INFINITY ? 0.f : exp2f(lse_own - mx);
          float sum = w_own;
#pragma unroll
          for (int e = 0; e < kHalf; ++e) o[e] *= w_own;
          for (int s2 = 0; s2 < pc.nslots; ++s2) {
            if (s2 == pc.slot) continue;
            const int64_t sl = (int64_t)s2 * p.sk_units + u;
            const float l = p.part_lse[sl * kBM + r];
            if (l == -INFINITY) continue;
            const float wt = exp2f(l - mx);
            sum += wt;
            const float* src = p.part_o + (sl * HD + col0) * kBM + r;
#pragma unroll
            for (int e = 0; e < kHalf; ++e) o[e] = fmaf(wt, src[e * kBM], o[e]);
          }
          const float inv = sum > 0.f ? 1.f / sum : 0.f;
#pragma unroll
          for (int e = 0; e < kHalf; ++e) o[e] *= inv;
        }
      }
      if (final_here) {
        // stage the bf16 tile in the canonical 128B-swizzled layout (64-column
        // halves of 128 rows x 128 B, like the Q tile) and TMA-store it; rows
        // past the last token are clipped by the tensor map
#pragma unroll
        for (int k = 0; k < kHalf / 8; ++k) {
          const int gcol = col0 + k * 8;
          const int hh = gcol >> 6, c16 = (gcol & 63) >> 3;
          uint4 v;
          v.x = pack_bf16x2(o[k * 8 + 0], o[k * 8 + 1]);
          v.y = pack_bf16x2(o[k * 8 + 2], o[k * 8 + 3]);
          v.z = pack_bf16x2(o[k * 8 + 4], o[k * 8 + 5]);
          v.w = pack_bf16x2(o[k * 8 + 6], o[k * 8 + 7]);
          *reinterpret_cast<uint4*>(sStage + hh * (kBM * 128) + r * 128 +
                                    ((c16 ^ (r & 7)) << 4)) = v;
        }
        fence_proxy_async_smem();
        named_bar_sync(2, 256);
        if (threadIdx.x == 0) ATTN_TRACE(180);
        if (threadIdx.x == 0) {
#pragma unroll
          for (int hh = 0; hh < HD / 64; ++hh)
            tma_store_3d(&tm_o, sStage + hh * (kBM * 128), hh * 64,
                         pack > 1 ? pc.head * pack : pc.head, tok(qt0));
          tma_store_commit();
          tma_store_wait_read();   // the staging tile is free again
        }
        named_bar_sync(2, 256);
        if (threadIdx.x == 0) ATTN_TRACE(181);
      }
      cw += my_tiles;
    }
  } else {
    shrink();  // warp 11
  }
  if (threadIdx.x == 0) ATTN_TRACE(182);

  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
  if (threadIdx.x == 0) ATTN_TRACE(4);
  if (p.num_splits == 1) launch_stamp_end(p.stamp);
}

// Deterministic split-KV combine: one warp per (query, head), splits in order.
template <int HD>
__global__ void __launch_bounds__(128)
    attn_combine_kernel(const float* __restrict__ part_o, const float* __restrict__ part_lse,
                        int num_splits, int rows, __nv_bfloat16* __restrict__ out,
                        unsigned long long* stamp) {
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
  if (stamp && lane == 0) atomicMax(stamp + 1, gtimer());  // per warp: rows may exit early
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
             int64_t rows, int64_t row_stride, int box_heads = 1) {
  EncodeTiledFn enc = get_encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return ASKV_ECUDA;
  }
  cuuint64_t dims[3] = {(cuuint64_t)head_dim, (cuuint64_t)heads, (cuuint64_t)rows};
  cuuint64_t strides[2] = {(cuuint64_t)head_stride * 2, (cuuint64_t)row_stride * 2};
  // box_heads > 1 (GQA packing): 128 / box_heads tokens x box_heads heads land as
  // 128 rows ordered (token, head), the same smem tile layout
  cuuint32_t box[3] = {64, (cuuint32_t)box_heads, (cuuint32_t)(128 / box_heads)};
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

// Pair two query tiles per CTA (M = 256 per K/V tile: half the K/V fill bytes
// per FLOP, the per-SM L2->SMEM fill rate being what bounds K3) only when one
// tile per CTA would need more than one wave of SMs; below that, pairing halves
// the CTA count and loses more than it saves (profiles/r01b_summary.md).
// ASKV_ATTN_PAIR=0/1 forces it off/on.
bool use_pairs(int q_tiles, int hq, int sms) {
  static int knob = -2;
  if (knob == -2) {
    const char* e = getenv("ASKV_ATTN_PAIR");
    knob = (e && e[0] == '1') ? 1 : (e && e[0] == '0') ? 0 : -1;
  }
  if (q_tiles < 2) return false;
  if (knob >= 0) return knob == 1;
  return q_tiles * hq > sms;
}

// GQA packing: when q-heads share a kv head, one CTA's
// 128 query rows are (token, q-head) pairs of a kv head, so each K/V tile
// feeds rows of every head of the group and a skinny prefill pads less (a
// 301-token tile set of 8 heads is 19 full tiles instead of 8 x 3 with a
// 45-row tail).  The group must divide the 128-row tile.  ASKV_ATTN_PACK=0
// turns it off.
int gqa_pack(int hq, int hkv) {
  static int knob = -1;
  if (knob < 0) {
    const char* e = getenv("ASKV_ATTN_PACK");
    knob = (e && e[0] == '0') ? 0 : 1;
  }
  const int g = hq / hkv;
  return (knob && g > 1 && g <= 16 && 128 % g == 0) ? g : 1;
}

// Split count minimising waves x (tiles per split + fixed per-CTA overhead).
// Split-KV policy, fitted to a B200 sweep (tools/kbench.py sweep): one CTA per
// SM at most (one wave), and at least 6 KV tiles per split so the per-CTA
// prologue / epilogue and the combine pass stay amortised (r01e sweep:
// (1000, 100, 40 heads) 20.5 us unsplit vs 23.5 us with 2 splits of 5 tiles).
// Stream-K schedule (attn_sk_kernel) is opt-in: ASKV_ATTN_SK=1.  Measured at
// the C3 shapes it loses to the (query tile, head[, split]) grid: its 148
// CTAs each pay the ~8 us per-CTA prologue / epilogue for ~10 KV tiles and
// the partials need a combine pass (profiles/r02_attn_stream_k.md).
bool use_sk() {
  static int knob = -1;
  if (knob < 0) {
    const char* e = getenv("ASKV_ATTN_SK");
    knob = (e && e[0] == '1') ? 1 : 0;
  }
  return knob == 1;
}

int choose_splits(int n_cached, int n_new, int hq, int sms, int hkv = 0) {
  if (hkv <= 0) hkv = hq;
  const int pack = gqa_pack(hq, hkv);
  const int q_tiles = (n_new * pack + kBM - 1) / kBM;
  // single-tile units: stream-K balances them over the SMs (one launch, no split)
  if (use_sk() && !(pack == 1 && use_pairs(q_tiles, hq, sms))) return 1;
  const int q_groups =
      pack == 1 && use_pairs(q_tiles, hq, sms) ? (q_tiles + 1) / 2 : q_tiles;
  const int kv_tiles = (n_cached + n_new + kBN - 1) / kBN;
  const int ctas = q_groups * (pack > 1 ? hkv : hq);
  int best = 1;
  for (int s = 2; s <= kMaxSplits; ++s) {
    const int tps = (kv_tiles + s - 1) / s;
    if (ctas * s > sms || tps < 6) break;
    if ((kv_tiles + tps - 1) / tps == s) best = s;
  }
  return best;
}

// Stream-K schedule on the host: the kernel's params, the CTA count and the
// partial slots the most-cut unit needs.
struct SkPlan {
  int ctas = 0, max_slots = 0;
};

void sk_plan(AttnParams& prm, int hkv, int sms, SkPlan& out) {
  const int q_rows = prm.pack > 1 ? prm.n_new * prm.pack : prm.n_new;
  const int qt = (q_rows + kBM - 1) / kBM;
  int per_head = 0;
  for (int q = 0; q < qt; ++q) per_head += unit_tiles(prm, q);
  const int heads = prm.pack > 1 ? hkv : prm.hq;
  prm.sk_tiles_head = per_head;
  prm.sk_q_tiles = qt;
  prm.sk_units = qt * heads;
  prm.sk_total = per_head * heads;
  // at least ceil(T_max / (kMaxSkSlots - 1)) tiles per CTA so no unit is cut
  // into more than kMaxSkSlots pieces
  const int t_max = unit_tiles(prm, qt - 1);
  const int min_per = (t_max + kMaxSkSlots - 2) / (kMaxSkSlots - 1);
  const int cap = prm.sk_total / min_per;
  static int knob = -1;   // ASKV_ATTN_SK_CTAS: CTA count override (measurement)
  if (knob < 0) {
    const char* e = getenv("ASKV_ATTN_SK_CTAS");
    knob = e ? atoi(e) : 0;
  }
  if (knob > 0) sms = knob;
  out.ctas = cap < sms ? (cap > 0 ? cap : 1) : sms;
  out.max_slots = 1;
  int ub = 0;
  for (int h = 0; h < heads; ++h)
    for (int q = 0; q < qt; ++q) {
      const int tu = unit_tiles(prm, q);
      const int ns = sk_owner(prm, ub + tu - 1, out.ctas) - sk_owner(prm, ub, out.ctas) + 1;
      if (ns > out.max_slots) out.max_slots = ns;
      ub += tu;
    }
}

size_t sk_workspace(int n_cached, int n_new, int hq, int hkv, int head_dim) {
  AttnParams prm{};
  prm.n_new = n_new;
  prm.n_cached = n_cached;
  prm.hq = hq;
  prm.group = hq / hkv;
  prm.pack = gqa_pack(hq, hkv);
  SkPlan plan;
  sk_plan(prm, hkv, sm_count(), plan);
  if (plan.max_slots <= 1) return 0;
  return (size_t)plan.max_slots * prm.sk_units * kBM * (head_dim + 1) * sizeof(float);
}

// Per-device arrival counters of the stream-K fixup (one int per unit).  The
// kernel leaves them zero (the last piece of a unit resets its counter), so
// they are zeroed once, at allocation, on a private stream (legal while the
// caller's stream is being captured).
constexpr int kSkMaxUnits = 1 << 16;
int* sk_counters() {
  static std::mutex mu;
  static std::map<int, int*> bufs;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  int*& b = bufs[dev];
  if (!b) {
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (cudaMalloc(&b, kSkMaxUnits * sizeof(int)) != cudaSuccess ||
        cudaMemsetAsync(b, 0, kSkMaxUnits * sizeof(int), st) != cudaSuccess ||
        cudaStreamSynchronize(st) != cudaSuccess)
      b = nullptr;
    cudaStreamDestroy(st);
  }
  return b;
}

template <int HD>
int launch_sk(const CUtensorMap& mq, const CUtensorMap& mk, const CUtensorMap& mv,
              const CUtensorMap& mvs, const CUtensorMap& mo, AttnParams prm, int hkv, void* ws,
              size_t ws_bytes, cudaStream_t stream) {
  SkPlan plan;
  sk_plan(prm, hkv, sm_count(), plan);
  ASKV_REQUIRE(prm.sk_units <= kSkMaxUnits, "prefill_attn: %d stream-K units > %d",
               prm.sk_units, kSkMaxUnits);
  const size_t slab = (size_t)prm.sk_units * kBM;
  const size_t need = plan.max_slots > 1
                          ? (size_t)plan.max_slots * slab * (HD + 1) * sizeof(float) : 0;
  ASKV_REQUIRE(need == 0 || (ws != nullptr && ws_bytes >= need),
               "prefill_attn: workspace %zu bytes < %zu needed (stream-K, %d slots)", ws_bytes,
               need, plan.max_slots);
  prm.part_o = static_cast<float*>(ws);
  prm.part_lse = need ? prm.part_o + (size_t)plan.max_slots * slab * HD : nullptr;
  prm.sk_cnt = sk_counters();
  if (!prm.sk_cnt) {
    set_error("prefill_attn: stream-K counters");
    return ASKV_ECUDA;
  }
  prm.num_splits = 1;  // the kernel stamps its own end (no combine pass)
  auto kern = attn_sk_kernel<HD>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         SkCfg<HD>::kSmemBytes);
    if (e != cudaSuccess) return cuda_status(e, "attn_sk smem attribute");
    attr = true;
  }
  kern<<<plan.ctas, SkCfg<HD>::kThreads, SkCfg<HD>::kSmemBytes, stream>>>(mq, mk, mv, mvs, mo,
                                                                          prm);
  return launch_status("attn_sk launch");
}

template <int HD>
int launch_attn(const void* q, const void* kv, int64_t kv_row_stride, int n_cached, int n_new,
                int hq, int hkv, float scale, void* out, void* ws, size_t ws_bytes,
                int splits, cudaStream_t stream, unsigned long long* stamp,
                const VSource* vsrc) {
  const int rows = n_cached + n_new;
  const int pack = gqa_pack(hq, hkv);
  CUtensorMap mq, mk, mv, mvs;
  int rc = make_map(&mq, q, HD, hq, HD, n_new, (int64_t)hq * HD, pack);
  if (!rc) rc = make_map(&mk, kv, HD, hkv, HD, rows, kv_row_stride);
  if (!rc)
    rc = make_map(&mv, static_cast<const __nv_bfloat16*>(kv) + (int64_t)hkv * HD, HD, hkv, HD,
                  rows, kv_row_stride);
  const bool use_vs = vsrc && vsrc->kind && vsrc->tiles > 0;
  if (!rc && use_vs)
    rc = make_map(&mvs, static_cast<const __nv_bfloat16*>(vsrc->base) + (int64_t)hkv * HD, HD,
                  hkv, HD, vsrc->rows, vsrc->row_elems);
  if (rc) return rc;
  if (!use_vs) mvs = mv;
  auto set_vs = [&](AttnParams& a) {
    a.v_src_tiles = use_vs ? vsrc->tiles : 0;
    a.v_src_row0 = use_vs ? vsrc->row0 : 0;
    a.v_blk_off = use_vs && vsrc->kind == 2 ? vsrc->blk_off : nullptr;
    a.v_row_elems = use_vs ? vsrc->row_elems : 1;
    a.v_layer_row = use_vs ? vsrc->layer_row : 0;
  };

  const int q_tiles = (n_new * pack + kBM - 1) / kBM;
  const bool paired = pack == 1 && use_pairs(q_tiles, hq, sm_count());
  const int q_groups = paired ? (q_tiles + 1) / 2 : q_tiles;
  const int kv_tiles = (rows + kBN - 1) / kBN;
  if (!paired && splits <= 1 && use_sk()) {
    AttnParams prm{};
    prm.n_new = n_new;
    prm.n_cached = n_cached;
    prm.hq = hq;
    prm.group = hq / hkv;
    prm.pack = pack;
    prm.scale_log2 = scale * 1.4426950408889634f;
    prm.out = static_cast<__nv_bfloat16*>(out);
    prm.stamp = stamp;
    set_vs(prm);
    CUtensorMap mo;
    rc = make_map(&mo, out, HD, hq, HD, n_new, (int64_t)hq * HD, pack);
    if (rc) return rc;
    return launch_sk<HD>(mq, mk, mv, mvs, mo, prm, hkv, ws, ws_bytes, stream);
  }
  const int tps = (kv_tiles + splits - 1) / splits;
  splits = (kv_tiles + tps - 1) / tps;
  AttnParams prm{};
  prm.n_new = n_new;
  prm.n_cached = n_cached;
  prm.hq = hq;
  prm.group = hq / hkv;
  prm.pack = pack;
  prm.num_splits = splits;
  prm.tiles_per_split = tps;
  prm.scale_log2 = scale * 1.4426950408889634f;
  prm.out = static_cast<__nv_bfloat16*>(out);
  prm.stamp = stamp;
  prm.part_o = nullptr;
  prm.part_lse = nullptr;
  set_vs(prm);
  if (splits > 1) {
    const size_t rows_qh = (size_t)n_new * hq;
    const size_t need = (size_t)splits * rows_qh * (HD + 1) * sizeof(float);
    ASKV_REQUIRE(ws != nullptr && ws_bytes >= need,
                 "prefill_attn: workspace %zu bytes < %zu needed for %d splits", ws_bytes, need,
                 splits);
    prm.part_o = static_cast<float*>(ws);
    prm.part_lse = prm.part_o + (size_t)splits * rows_qh * HD;
  }
  dim3 grid(q_groups, pack > 1 ? hkv : hq, splits);
  if (paired) {
    auto kern = attn_fwd_kernel<HD, true>;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           Cfg<HD, true>::kSmemBytes);
      if (e != cudaSuccess) return cuda_status(e, "attn smem attribute");
      attr = true;
    }
    VarJobs none;
    none.n = 0;
    kern<<<grid, Cfg<HD, true>::kThreads, Cfg<HD, true>::kSmemBytes, stream>>>(mq, mk, mv, mvs,
                                                                                prm, none);
  } else {
    auto kern = attn_fwd_kernel<HD, false>;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           Cfg<HD, false>::kSmemBytes);
      if (e != cudaSuccess) return cuda_status(e, "attn smem attribute");
      attr = true;
    }
    VarJobs none;
    none.n = 0;
    kern<<<grid, Cfg<HD, false>::kThreads, Cfg<HD, false>::kSmemBytes, stream>>>(mq, mk, mv,
                                                                                 mvs, prm, none);
  }
  rc = launch_status("attn_fwd launch");
  if (rc || splits == 1) return rc;
  const int rows_qh = n_new * hq;
  attn_combine_kernel<HD><<<(rows_qh + 3) / 4, 128, 0, stream>>>(
      prm.part_o, prm.part_lse, splits, rows_qh, static_cast<__nv_bfloat16*>(out), stamp);
  return launch_status("attn_combine launch");
}

template <int HD>
int launch_varlen(const VarlenBatch& b, cudaStream_t stream, unsigned long long* stamp) {
  const int hq = b.hq, hkv = b.hkv;
  const int pack = gqa_pack(hq, hkv);
  const int heads = pack > 1 ? hkv : hq;
  int q_tot = 0, kv_tot = 0;
  for (int i = 0; i < b.n; ++i) {
    q_tot = std::max(q_tot, b.q_row0[i] + b.n_new[i]);
    kv_tot = std::max(kv_tot, b.kv_row0[i] + b.n_cached[i] + b.n_new[i]);
  }
  CUtensorMap mq, mk, mv, mvs;
  int rc = make_map(&mq, b.q, HD, hq, HD, q_tot, (int64_t)hq * HD, pack);
  if (!rc) rc = make_map(&mk, b.kv, HD, hkv, HD, kv_tot, b.kv_row_stride);
  if (!rc)
    rc = make_map(&mv, static_cast<const __nv_bfloat16*>(b.kv) + (int64_t)hkv * HD, HD, hkv, HD,
                  kv_tot, b.kv_row_stride);
  const bool use_vs = b.vsrc_base != nullptr;
  if (!rc && use_vs)
    rc = make_map(&mvs, static_cast<const __nv_bfloat16*>(b.vsrc_base) + (int64_t)hkv * HD, HD,
                  hkv, HD, b.vsrc_rows, b.vsrc_row_elems);
  if (rc) return rc;
  if (!use_vs) mvs = mv;
  AttnParams prm{};
  prm.hq = hq;
  prm.group = hq / hkv;
  prm.pack = pack;
  prm.num_splits = 1;
  prm.tiles_per_split = 1 << 20;
  prm.scale_log2 = b.scale * 1.4426950408889634f;
  prm.stamp = stamp;
  prm.v_row_elems = use_vs ? b.vsrc_row_elems : 1;
  // Pair two query tiles of a job per CTA when the batch has more than a wave
  // of query tiles (the usual case): each K/V tile feeds 256 query rows and
  // the per-CTA prologue / epilogue is paid once per two tiles.  A job's odd
  // last tile runs alone in the paired kernel (its CTA-uniform unpaired mode).
  int q_tiles_all = 0;
  for (int i = 0; i < b.n; ++i) q_tiles_all += (b.n_new[i] * pack + kBM - 1) / kBM;
  const bool pair = pack == 1 && use_pairs(q_tiles_all, heads, sm_count());
  const int qt_per_cta = pair ? 2 : 1;
  auto kern = pair ? attn_fwd_kernel<HD, true> : attn_fwd_kernel<HD, false>;
  const int smem = pair ? Cfg<HD, true>::kSmemBytes : Cfg<HD, false>::kSmemBytes;
  static bool attr[2] = {false, false};
  if (!attr[pair]) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return cuda_status(e, "attn smem attribute");
    attr[pair] = true;
  }
  // jobs in descending KV length: the longest CTAs start first and the last
  // wave is made of short ones (longest-processing-time-first)
  int order[kMaxVarJobs];
  for (int i0 = 0; i0 < b.n; i0 += kMaxVarJobs) {   // <= kMaxVarJobs jobs per launch
    VarJobs vj;
    vj.n = std::min(kMaxVarJobs, b.n - i0);
    for (int k = 0; k < vj.n; ++k) order[k] = i0 + k;
    std::stable_sort(order, order + vj.n, [&](int x, int y) {
      return b.n_cached[x] + b.n_new[x] > b.n_cached[y] + b.n_new[y];
    });
    int ctas = 0;
    for (int k = 0; k < vj.n; ++k) {
      const int i = order[k];
      VarJob& J = vj.j[k];
      J.n_new = b.n_new[i];
      J.n_cached = b.n_cached[i];
      J.q_row0 = b.q_row0[i];
      J.kv_row0 = b.kv_row0[i];
      J.cta0 = ctas;
      J.q_groups = (b.n_new[i] * pack + kBM * qt_per_cta - 1) / (kBM * qt_per_cta);
      J.v_src_tiles = use_vs ? b.v_src_tiles[i] : 0;
      J.v_blk_off = use_vs ? b.v_blk_off[i] : nullptr;
      J.v_layer_row = b.v_layer_row;
      J.out = static_cast<__nv_bfloat16*>(b.out[i]);
      ctas += J.q_groups * heads;
    }
    kern<<<ctas, pair ? Cfg<HD, true>::kThreads : Cfg<HD, false>::kThreads, smem, stream>>>(
        mq, mk, mv, mvs, prm, vj);
    rc = launch_status("attn_fwd varlen launch");
    if (rc) return rc;
  }
  return ASKV_OK;
}

}  // namespace
}  // namespace askv

using namespace askv;

extern "C" int askv_attn_num_splits(int n_cached, int n_new, int n_heads, int sms) {
  if (n_new <= 0 || n_heads <= 0 || n_cached < 0) return 1;
  return choose_splits(n_cached, n_new, n_heads, sms > 0 ? sms : sm_count());
}

extern "C" int askv_attn_num_splits_gqa(int n_cached, int n_new, int n_heads, int n_kv_heads,
                                        int sms) {
  if (n_new <= 0 || n_heads <= 0 || n_cached < 0 || n_kv_heads <= 0 ||
      n_heads % n_kv_heads)
    return 1;
  return choose_splits(n_cached, n_new, n_heads, sms > 0 ? sms : sm_count(), n_kv_heads);
}

extern "C" size_t askv_attn_workspace_bytes_gqa(int n_cached, int n_new, int n_heads,
                                                int n_kv_heads, int head_dim, int num_splits) {
  if (n_new <= 0 || n_heads <= 0 || n_kv_heads <= 0 || n_heads % n_kv_heads) return 0;
  const int s = num_splits > 0
                    ? num_splits
                    : choose_splits(n_cached, n_new, n_heads, sm_count(), n_kv_heads);
  if (s > 1) return (size_t)s * n_new * n_heads * (head_dim + 1) * sizeof(float);
  const int pack = gqa_pack(n_heads, n_kv_heads);
  const int q_tiles = (n_new * pack + kBM - 1) / kBM;
  if (!use_sk() || (pack == 1 && use_pairs(q_tiles, n_heads, sm_count()))) return 0;
  return sk_workspace(n_cached, n_new, n_heads, n_kv_heads, head_dim);
}

// Without the kv-head count: the largest need over every GQA grouping of n_heads.
extern "C" size_t askv_attn_workspace_bytes(int n_cached, int n_new, int n_heads,
                                            int head_dim, int num_splits) {
  size_t best = 0;
  for (int hkv = 1; hkv <= n_heads; ++hkv) {
    if (n_heads % hkv) continue;
    const size_t b =
        askv_attn_workspace_bytes_gqa(n_cached, n_new, n_heads, hkv, head_dim, num_splits);
    if (b > best) best = b;
  }
  return best;
}

extern "C" int askv_prefill_attn(const void* q, const void* kv, int64_t kv_row_stride,
                                 int n_cached, int n_new, int n_heads, int n_kv_heads,
                                 int head_dim, float scale, void* out, void* workspace,
                                 size_t workspace_bytes, int num_splits, void* stream) {
  clear_error();
  return askv::prefill_attn_stamped(q, kv, kv_row_stride, n_cached, n_new, n_heads, n_kv_heads,
                                    head_dim, scale, out, workspace, workspace_bytes, num_splits,
                                    stream, nullptr);
}

int askv::prefill_attn_stamped(const void* q, const void* kv, int64_t kv_row_stride,
                               int n_cached, int n_new, int n_heads, int n_kv_heads,
                               int head_dim, float scale, void* out, void* workspace,
                               size_t workspace_bytes, int num_splits, void* stream,
                               unsigned long long* stamp, const VSource* vsrc) {
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
  int splits = num_splits > 0 ? num_splits
                              : choose_splits(n_cached, n_new, n_heads, sm_count(), n_kv_heads);
  if (head_dim == 128)
    return launch_attn<128>(q, kv, kv_row_stride, n_cached, n_new, n_heads, n_kv_heads, scale,
                            out, workspace, workspace_bytes, splits, (cudaStream_t)stream, stamp,
                            vsrc);
  return launch_attn<64>(q, kv, kv_row_stride, n_cached, n_new, n_heads, n_kv_heads, scale, out,
                         workspace, workspace_bytes, splits, (cudaStream_t)stream, stamp, vsrc);
}

int askv::prefill_attn_varlen(const VarlenBatch& b, void* stream, unsigned long long* stamp) {
  ASKV_REQUIRE(b.n >= 1 && b.hq > 0 && b.hkv > 0 && b.hq % b.hkv == 0,
               "prefill_attn_varlen: bad batch");
  ASKV_REQUIRE(b.head_dim == 64 || b.head_dim == 128, "prefill_attn_varlen: head_dim %d",
               b.head_dim);
  for (int i = 0; i < b.n; ++i)
    ASKV_REQUIRE(b.n_new[i] > 0 && b.n_cached[i] >= 0 && b.out[i],
                 "prefill_attn_varlen: job %d", i);
  if (b.head_dim == 128) return launch_varlen<128>(b, (cudaStream_t)stream, stamp);
  return launch_varlen<64>(b, (cudaStream_t)stream, stamp);
}
