// build.cu — GPU CSR -> HRPB builder, bit-identical to the oracle.
//
// Paper: Alg. "CSR to HRPB Phase1/Phase2" runs on the host with OpenMP over panel
// chunks and prefix sums; §"HRPB Sparse Matrix Data structure" defines the output.
// B200 design: no host round trip until the end; outputs are allocated at
// upper bounds computable from (M, nnz), so the pipeline is
//   k_wclassify            (panels the warp path cannot take: > wcap entries or a column span wider than its
//                           bitmap -> listed)
//   k_count / k_count_big  (B1 + B3 counting per listed panel by a CTA / hub CTAs: ranks q of every entry,
//                           patterns kept in scratch, nact, nblk, bytes; CSR validation)
//   k_wbuild               (warp per panel, ticket-ordered: B1 + B3 bitmap ranking and patterns, then the
//                           single-pass decoupled look-back scans B2 blockedRowPtr / B4 panel byte offsets over
//                           ALL panels, then B3 + B4 + B5 emission of its panel)
//   k_emit                 (B3 + B4 + B5 for listed panels: activeCols with sentinel K, sizePtr, HRPB-v1
//                           headers, patterns, values in brick-CSC / row-major order)
//   k_finalize             (NUM_BLKS, byte total, status) -> one 32-byte D2H read + sync.
// Listed panel p keeps its brick patterns between the two passes in a scratch region addressed from its
// first entry offset, base(p) = floor(e0 * nbk / tk) + 2 p nbk, which never overlaps the next panel's.
#include <cstdio>

#include <cub/block/block_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "internal.h"

namespace hrpb {

enum : uint32_t {
  ST_RP0 = 1u,        // row_ptr[0] != 0
  ST_RP_MONO = 2u,    // row_ptr decreasing
  ST_COL_RANGE = 4u,  // column outside [0, K)
  ST_COL_ORDER = 8u,  // columns not strictly increasing within a row
  ST_NNZ = 16u,       // row_ptr[M] != nnz
};

constexpr int kSmallThreads = 128;
constexpr int kSmallCap = 2048;      // entries per panel handled in shared memory
#ifndef HRPB_3P_MIN_PANELS
#define HRPB_3P_MIN_PANELS 196608
#endif
constexpr int64_t kThreePhaseMinPanels = HRPB_3P_MIN_PANELS;  // k_wbuild count / scan / emit from this many panels
constexpr int kSpanWords = 512;      // bitmap ranking when the panel's column span <= 16384
constexpr int kBigThreads = 512;
#ifndef HRPB_BIG_CTAS_PER_SM
#define HRPB_BIG_CTAS_PER_SM 2  // hub CTAs per SM (each with its own column bitmap scratch, ~1 MB at K = 4M)
#endif
#ifndef HRPB_HUB_EMIT
#define HRPB_HUB_EMIT 16384
#endif
#ifndef HRPB_HUB_CHUNK
#define HRPB_HUB_CHUNK 4096
#endif
constexpr int64_t kHubEmit = HRPB_HUB_EMIT;    // listed panels above this many entries: values by k_emit_hubvals
constexpr int64_t kHubChunk = HRPB_HUB_CHUNK;  // entries per k_emit_hubvals work item  // listed panels with more entries get their values scattered by all CTAs
constexpr int kEmitThreads = 128;

// ------------------------------------------------------------------ block-wide helpers
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* total, uint32_t* sh /*[NT/32+1]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (warp == 0) {
    uint32_t w = lane < NT / 32 ? sh[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) sh[lane] = w;  // inclusive warp totals
  }
  __syncthreads();
  uint32_t base = warp ? sh[warp - 1] : 0;
  uint32_t tot = sh[NT / 32 - 1];
  __syncthreads();
  if (total) *total = tot;
  return base + x - v;
}

template <int NT>
__device__ __forceinline__ void block_minmax(int32_t& mn, int32_t& mx, int32_t* sh /*[2*NT/32]*/) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if (lane == 0) { sh[warp] = mn; sh[NT / 32 + warp] = mx; }
  __syncthreads();
  mn = sh[0];
  mx = sh[NT / 32];
  for (int w = 1; w < NT / 32; ++w) { mn = min(mn, sh[w]); mx = max(mx, sh[NT / 32 + w]); }
  __syncthreads();
}

// Row pointers of panel p -> shared memory, clamped to [0, nnz] and repaired to be monotone (memory
// safety on invalid input); a decreasing raw row_ptr is flagged in *status. One warp, one sync.
__device__ __forceinline__ void load_panel_rows(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int tm,
                                                int64_t p, int64_t* s_rp, uint32_t* status) {
  const int64_t r0 = p * tm;
  const int nrows = (int)min((int64_t)tm, M - r0);
  __syncthreads();  // s_rp may still be read by the previous panel iteration
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    int64_t carry = 0;
    bool bad = false;
    for (int base = 0; base <= nrows; base += 32) {
      const int i = base + lane;
      const int64_t raw = i <= nrows ? rp[r0 + i] : INT64_MAX;
      int64_t prev = __shfl_up_sync(0xffffffffu, raw, 1);
      if (lane == 0) prev = base == 0 ? raw : carry;
      if (i <= nrows && raw < prev) bad = true;
      int64_t v = raw < 0 ? 0 : (raw > nnz ? nnz : raw);
      if (i > nrows) v = 0;
      for (int o = 1; o < 32; o <<= 1) {  // inclusive running max (monotone repair)
        const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v = max(v, y);
      }
      if (base > 0) v = max(v, s_rp[base - 1]);
      if (i <= nrows) s_rp[i] = v;
      carry = __shfl_sync(0xffffffffu, raw, 31);
      __syncwarp();
    }
    if (__any_sync(0xffffffffu, bad) && status && lane == 0) atomicOr(status, ST_RP_MONO);
  }
  __syncthreads();
}

// local row of panel entry e (s_rp[r] <= e < s_rp[r+1]); binary search over <= 129 row pointers
__device__ __forceinline__ int row_of(const int64_t* s_rp, int nrows, int64_t e) {
  int lo = 0, hi = nrows - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (s_rp[mid] <= e) lo = mid;
    else hi = mid - 1;
  }
  return lo;
}

__device__ __forceinline__ int64_t pat_base(int64_t e0, int64_t p, int nbk, int tk) {
  return e0 * nbk / tk + 2 * p * nbk;
}

// ------------------------------------------------------------------ warp-level helpers
__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t* total) {
  const int lane = threadIdx.x & 31;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (total) *total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

// Warp-wide version of load_panel_rows (no CTA barrier): clamped, monotone-repaired row pointers.
__device__ __forceinline__ void warp_panel_rows(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int tm,
                                                int64_t p, int64_t* s_rp, uint32_t* status) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = p * tm;
  const int nrows = (int)min((int64_t)tm, M - r0);
  int64_t carry_raw = 0, carry_v = 0;
  bool bad = false;
  for (int base = 0; base <= nrows; base += 32) {
    const int i = base + lane;
    const int64_t raw = i <= nrows ? rp[r0 + i] : INT64_MAX;
    int64_t prev = __shfl_up_sync(0xffffffffu, raw, 1);
    if (lane == 0) prev = base == 0 ? raw : carry_raw;
    if (i <= nrows && raw < prev) bad = true;
    int64_t v = i <= nrows ? (raw < 0 ? 0 : (raw > nnz ? nnz : raw)) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v = max(v, y);
    }
    v = max(v, carry_v);
    if (i <= nrows) s_rp[i] = v;
    carry_raw = __shfl_sync(0xffffffffu, raw, 31);
    carry_v = __shfl_sync(0xffffffffu, v, 31);
  }
  if (__any_sync(0xffffffffu, bad) && status && lane == 0) atomicOr(status, ST_RP_MONO);
  __syncwarp();
}

// ------------------------------------------------------------------ warp-per-panel path (most panels)
// One warp owns one panel with at most kWCap entries whose column span fits the kWBmWords-word bitmap
// (c1, c2a/c2b at every TM). k_wbuild ranks, scans and emits in one pass, so no per-entry rank or per-brick
// pattern array goes through HBM and the CSR is read once (plus L1 re-reads).
//   ranks ("active_cols = uniq(...)", R23): bitmap over [mn, mn + span) + popcount prefix per word
//   rows: a per-panel u8 row map in shared memory, each lane filling its own row (no per-entry search)
//   patterns (P:L132 fill_brick_nnz_pattern; bit = (r % 16) * 4 + q % 4, R3): 32-bit shared atomicOr
// Panels that do not fit go to the CTA / hub paths (k_count, k_count_big, k_emit), listed by k_wclassify.
constexpr int kWCap = 1024;       // entries per panel on the warp path (TM = 128: 512, see wcap)
constexpr int kWBmWords = 256;    // bitmap words: column span <= 8192
constexpr int kWNarrow = 768;     // spans below this mark columns in a byte map (plain stores, no atomics)
constexpr int kWByteMap = 256;    // byte offset of the byte map (after the <= 24 bitmap words it turns into)
static_assert(kWByteMap >= kWNarrow / 8 && kWByteMap + kWNarrow <= 4 * kWBmWords, "byte map inside the bitmap area");
// brick slots held at once (patterns are built per chunk of blocks): 16 blocks' worth, at most 128 slots — the
// per-warp shared memory bounds the resident warps of this latency-bound kernel (measured on c2a: 256 slots
// 0.333 / 0.427 ms at TM = 64 / 16, 128 slots 0.322 / 0.401, 64 slots 0.407 (two chunks) / 0.377)
__host__ __device__ constexpr int wslots(int tm, int tk) {
  return 16 * (tk / HRPB_BRICK_K) * (tm / HRPB_BRICK_M) < 128 ? 16 * (tk / HRPB_BRICK_K) * (tm / HRPB_BRICK_M)
                                                                : 128;
}
#ifndef HRPB_WWARPS
#define HRPB_WWARPS 4
#endif
constexpr int kWWarps = HRPB_WWARPS;  // warps per CTA (k_wclassify, k_wbuild)
constexpr int kB = 4;             // entries per lane per round in the warp-path entry loops
#ifndef HRPB_WB_MINB
#define HRPB_WB_MINB 5            // k_wbuild CTAs per SM the register allocation must allow (shared memory: 5)
#endif

struct WarpLayout {  // per-warp shared memory (bytes), depends on tm/tk only
  int slots;         // brick slots per block chunk = wslots (a chunk is wslots / nbk blocks)
  int off_pre, off_row, off_q, off_pat, off_soff, off_vbase, off_stage, bytes;
};
constexpr int kWSortCap = 256;  // wide-span panels with <= 256 entries: warp bitonic sort ranking
static_assert(kWSortCap * 8 <= 2 * kWBmWords * 4, "sort keys alias the bitmap + prefix words");
__host__ __device__ constexpr int wcap(int tm, int) { return tm == 16 ? kWCap / 2 : kWCap; }
__host__ __device__ inline WarpLayout warp_layout(int tm, int tk) {  // (also used by the host launcher)
  const int nbk = (tk / HRPB_BRICK_K) * (tm / HRPB_BRICK_M);
  WarpLayout L;
  const int cap = wcap(tm, tk);
  L.slots = wslots(tm, tk);
  L.off_pre = kWBmWords * 4;
  L.off_row = L.off_pre + kWBmWords * 4;                    // u8 row of each entry
  L.off_q = L.off_row + cap;                                // u16 rank of each entry
  L.off_pat = (L.off_q + 2 * cap + 7) & ~7;
  const int sl = (L.slots / nbk) * (nbk + 1);                // slots with one pad slot per block (bank skew)
  L.off_soff = L.off_pat + sl * 8;
  L.off_vbase = (L.off_soff + sl * 2 + 7) & ~7;
  L.off_stage = (L.off_vbase + (L.slots / nbk) * 8 + 15) & ~15;  // staged col_idx, later the values
  L.bytes = L.off_stage + 4 * (cap + 8);
  return L;
}

struct WarpPanel {
  int64_t p, e0;
  int E, nrows;
  int64_t Eall;     // entries of the panel (E is clamped to kWCap + 1)
  int32_t mn;
  uint32_t nact, nblk;
  bool sorted;      // rank by warp sort (column span wider than the bitmap, E <= kWSortCap)
  bool patterns_done;  // the rank pass also set the brick patterns (all blocks in one slot chunk)
  int nbw;          // bitmap words in use: ceil(span / 32) <= kWNarrow / 32 (byte-map path) or kWBmWords
  uint32_t st[4];   // row starts of rows lane + 32k (entry index relative to e0), valid for 1 <= r < nrows
};

// Loads the panel's row pointers (clamped, monotone-repaired; ST_RP_MONO on a decreasing row_ptr) into
// per-lane registers and decides whether the warp path takes the panel: E <= kWCap and the column span
// (first / last entries of the sorted rows) fits the bitmap. Returns false otherwise (warp-uniform).
template <int tm, int tk>
__device__ __forceinline__ bool warp_panel_rows(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int64_t p,
                                                WarpPanel& w, uint32_t* status) {
  const int lane = threadIdx.x & 31;
  const int64_t r0 = p * tm;
  const int nrows = (int)min((int64_t)tm, M - r0);
  int64_t carry = INT64_MIN;
  bool bad = false;
  constexpr int KV = tm / 32 + 1;  // row-pointer registers per lane
  int64_t v[KV + 1];  // rp[r0 + lane + 32k] (the last used one covers rp[r0 + nrows]); v[KV] = 0 pad
  const int nk = nrows / 32 + 1;
  v[KV] = 0;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    v[k] = 0;
    if (k >= nk) continue;  // warp-uniform
    const int i = lane + 32 * k;
    const bool in = i <= nrows;
    const int64_t raw = in ? rp[r0 + i] : INT64_MAX;
    int64_t prev = __shfl_up_sync(0xffffffffu, raw, 1);
    if (lane == 0) prev = k == 0 ? raw : carry;
    if (in && raw < prev) bad = true;
    int64_t x = in ? (raw < 0 ? 0 : (raw > nnz ? nnz : raw)) : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x = max(x, y);
    }
    if (k > 0) x = max(x, __shfl_sync(0xffffffffu, v[k - 1], 31));
    v[k] = x;
    carry = __shfl_sync(0xffffffffu, raw, 31);
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0 && status) atomicOr(status, ST_RP_MONO);
  const int last_k = nrows >> 5, last_l = nrows & 31;
  int64_t e1 = 0, e0 = 0;
#pragma unroll
  for (int k = 0; k < KV; ++k) {
    const int64_t t = __shfl_sync(0xffffffffu, v[k], last_l);
    if (k == last_k) e1 = t;
  }
  e0 = __shfl_sync(0xffffffffu, v[0], 0);
  w.p = p;
  w.e0 = e0;
  w.nrows = nrows;
  const int64_t E = e1 - e0;
  w.Eall = E;
  w.E = (int)min(E, (int64_t)kWCap + 1);
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int r = lane + 32 * k;
    w.st[k] = (k < KV && r >= 1 && r < nrows) ? (uint32_t)(v[k < KV ? k : 0] - e0) : 0xFFFFFFFFu;
  }
  return E <= wcap(tm, tk);
}

// Column span of a panel from the first and last entry of each (sorted) row; col(i) returns the column of panel
// entry e0 + i. Decides the ranking method (bitmap, or warp sort for small wide panels) and whether the warp
// path takes the panel at all.
template <int tm, typename GetCol>
__device__ __forceinline__ bool warp_panel_span(WarpPanel& w, GetCol col) {
  const int lane = threadIdx.x & 31;
  int32_t mn = INT32_MAX, mx = INT32_MIN;
#pragma unroll
  for (int k = 0; k < (tm + 31) / 32; ++k) {
    const int r = lane + 32 * k;
    const uint32_t nx_same = __shfl_sync(0xffffffffu, w.st[k], (lane + 1) & 31);
    const uint32_t nx_next = __shfl_sync(0xffffffffu, w.st[k < 3 ? k + 1 : 3], 0);
    if (r < w.nrows) {
      const uint32_t beg = r == 0 ? 0u : w.st[k];
      const uint32_t end = r + 1 >= w.nrows ? (uint32_t)w.E : (lane == 31 ? nx_next : nx_same);
      if (end > beg) {
        mn = min(mn, col(beg));
        mx = max(mx, col(end - 1));
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  w.mn = mn;
  w.sorted = false;
  w.nbw = kWBmWords;
  if (w.E == 0) return true;
  if ((int64_t)mx - (int64_t)mn < kWNarrow) w.nbw = (int)(((int64_t)mx - (int64_t)mn) / 32) + 1;
  if ((int64_t)mx - (int64_t)mn < 32 * kWBmWords) return true;
  w.sorted = true;
  return w.E <= kWSortCap;
}

// Stages 4-byte elements [e0, e0 + E) of a CSR array into shared memory with cp.async (one latency for the
// whole panel): 16-B copies from the 16-B aligned window around e0 (src-size clamps at nnz) when the array base
// is 16-B aligned, else 4-B copies. Commits one cp.async group; returns the offset of e0 in the window.
__device__ __forceinline__ int warp_stage(const void* __restrict__ base, int64_t nnz, int64_t e0, int E, uint8_t* dst,
                                          bool al16) {
  const int lane = threadIdx.x & 31;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(base);
  int shift = 0;
  if (al16) {
    shift = (int)(e0 & 3);
    const int64_t a0 = e0 - shift;
    const int nch = (shift + E + 3) >> 2;
    for (int c = lane; c < nch; c += 32) {
      const int64_t idx = a0 + 4 * c;
      const uint32_t bytes = idx + 4 <= nnz ? 16u : (idx < nnz ? (uint32_t)(nnz - idx) * 4u : 0u);
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst + 16 * c)),
                   "l"(src + (idx < nnz ? idx : 0)), "r"(bytes) : "memory");
    }
  } else {
    for (int i = lane; i < E; i += 32)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst + 4 * i)), "l"(src + e0 + i)
                   : "memory");
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  return shift;
}
__device__ __forceinline__ void warp_stage_wait() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
  __syncwarp();
}

// row map: srow[i] = local row of panel entry e0 + i; lane r fills its own row's entries (row ends from the
// neighbouring lane's start; empty rows write nothing)
template <int tm>
__device__ __forceinline__ void warp_row_map(const WarpPanel& w, uint8_t* srow) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < (tm + 31) / 32; ++k) {
    if (32 * k >= w.nrows) break;  // warp-uniform
    const int r = lane + 32 * k;
    const uint32_t nx_same = __shfl_sync(0xffffffffu, w.st[k], (lane + 1) & 31);
    const uint32_t nx_next = __shfl_sync(0xffffffffu, w.st[k < 3 ? k + 1 : 3], 0);
    if (r < w.nrows) {
      const uint32_t beg = r == 0 ? 0u : w.st[k];
      const uint32_t end = r + 1 >= w.nrows ? (uint32_t)w.E : (lane == 31 ? nx_next : nx_same);
      for (uint32_t e = beg; e < end; ++e) srow[e] = (uint8_t)r;
    }
  }
  __syncwarp();
}

// Ranks (bitmap + prefix) and brick patterns of a warp-path panel into the warp's shared memory; validates
// columns (ST_COL_RANGE) and in-row order (ST_COL_ORDER). Returns false if the brick slots of the
// panel exceed the layout (then the panel is listed for the CTA path).
template <int tm, int tk>
__device__ __forceinline__ bool warp_panel_rank(const int32_t* __restrict__ scol, int64_t K, WarpPanel& w,
                                                uint8_t* my, const WarpLayout& L, uint32_t* status) {
  const int lane = threadIdx.x & 31;
  uint32_t* bm = reinterpret_cast<uint32_t*>(my);
  uint32_t* pre = reinterpret_cast<uint32_t*>(my + L.off_pre);
  uint64_t* keys = reinterpret_cast<uint64_t*>(my);  // sort path (aliases bm + pre)
  uint8_t* srow = my + L.off_row;
  uint16_t* sq = reinterpret_cast<uint16_t*>(my + L.off_q);
  const bool sorted = w.sorted;
  const int nbw = w.nbw;
  const bool narrow = !sorted && nbw < kWBmWords;
  w.patterns_done = false;
  uint8_t* bmap = my + kWByteMap;  // narrow spans: one byte per column of [mn, mn + 32 nbw)
  if (narrow) {
    for (int i = lane; i < 8 * nbw; i += 32) reinterpret_cast<uint32_t*>(bmap)[i] = 0u;
  } else if (!sorted) {
#pragma unroll
    for (int i = 0; i < kWBmWords / 32; ++i) bm[lane + 32 * i] = 0u;
  }
  warp_row_map<tm>(w, srow);
  const int E = w.E;
  const int32_t mn = w.mn;
  bool bad_range = false, bad_order = false;
  // Loops over the entries run kB entries per lane per round with every shared load of the round issued before
  // its stores (generic pointers: the compiler cannot move the next entry's loads above a store itself).
  for (int c0 = 0; c0 < E; c0 += 32 * kB) {  // pass 1: validation + bitmap bits (or sort keys)
    int rr[kB], rp1[kB];
    int32_t cc[kB], cp1[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = c0 + 32 * u + lane;
      const bool in = i < E;
      rr[u] = in ? srow[i] : 0;
      cc[u] = in ? scol[i] : 0;
      rp1[u] = in && i > 0 ? srow[i - 1] : -1;
      cp1[u] = in && i > 0 ? scol[i - 1] : 0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = c0 + 32 * u + lane;
      if (i >= E) continue;
      const int r = rr[u];
      const int32_t c = cc[u];
      // in-row order against the previous entry, read from shared memory (no shuffle chain)
      if (rp1[u] == r && cp1[u] >= c) bad_order = true;
      const uint32_t off = (uint32_t)(c - mn);
      if (c < 0 || c >= K) bad_range = true;
      if (sorted) {
        keys[i] = ((uint64_t)(uint32_t)c << 32) | (uint32_t)i;
      } else if (off >= 32u * nbw) {
        bad_order = true;  // only an unsorted row can leave [mn, mx]
        sq[i] = 0xFFFFu;
      } else {
        // byte map: same-word stores from many lanes cost one wavefront; bitmap atomics on the few words of a
        // banded panel serialised ~16-way (ncu: 8.7M of k_wbuild's 50M shared wavefronts)
        if (narrow) bmap[off] = 1;
        else atomicOr(&bm[off >> 5], 1u << (off & 31));
        sq[i] = (uint16_t)off;  // column offset, turned into the rank below (no second global load)
      }
    }
  }
  const bool any_range = __any_sync(0xffffffffu, bad_range), any_order = __any_sync(0xffffffffu, bad_order);
  if (status && lane == 0) {
    if (any_range) atomicOr(status, ST_COL_RANGE);
    if (any_order) atomicOr(status, ST_COL_ORDER);
  }
  __syncwarp();
  uint32_t nact;
  if (narrow) {  // byte map -> bitmap words (lane l: columns [32 l, 32 l + 32)) + popcount prefix
    uint32_t word = 0;
    if (lane < nbw) {
      const uint4* src = reinterpret_cast<const uint4*>(bmap + 32 * lane);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint4 v = src[h];
        const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)  // bytes are 0 / 1: gather bits 0, 8, 16, 24 into a nibble
          word |= ((x[k] | (x[k] >> 7) | (x[k] >> 14) | (x[k] >> 21)) & 0xFu) << (16 * h + 4 * k);
      }
    }
    const uint32_t run = warp_excl_scan((uint32_t)__popc(word), &nact);
    if (lane < nbw) { bm[lane] = word; pre[lane] = run; }
    __syncwarp();
  }
  if (!sorted) {
    if (!narrow) {
      constexpr int kW = kWBmWords / 32;
      uint32_t cnt[kW], sum = 0;
#pragma unroll
      for (int i = 0; i < kW; ++i) { cnt[i] = __popc(bm[lane * kW + i]); sum += cnt[i]; }
      uint32_t run = warp_excl_scan(sum, &nact);
#pragma unroll
      for (int i = 0; i < kW; ++i) { pre[lane * kW + i] = run; run += cnt[i]; }
      __syncwarp();
    }
    // all blocks' patterns fit the slot array (one chunk): set the brick pattern bits in the rank loop itself
    constexpr int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
    constexpr int tk_sh = tk == 16 ? 4 : 5;
    const bool fuse = (nact + tk - 1) / tk <= (uint32_t)(wslots(tm, tk) / nbk);
    uint32_t* pat32 = reinterpret_cast<uint32_t*>(my + L.off_pat);
    if (fuse) {
      for (int i = lane; i < 2 * (int)((nact + tk - 1) / tk) * (nbk + 1); i += 32) pat32[i] = 0u;
      __syncwarp();
    }
    for (int c0 = 0; c0 < E; c0 += 32 * kB) {  // ranks: popcount prefix of the lower bits (R23: ascending columns)
      uint32_t off[kB], qq[kB];
      int ra[kB];
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        off[u] = c0 + 32 * u + lane < E ? sq[c0 + 32 * u + lane] : 0xFFFFu;
        ra[u] = fuse && c0 + 32 * u + lane < E ? srow[c0 + 32 * u + lane] : 0;
      }
#pragma unroll
      for (int u = 0; u < kB; ++u)
        qq[u] = off[u] < 32u * nbw ? pre[off[u] >> 5] + __popc(bm[off[u] >> 5] & ((1u << (off[u] & 31)) - 1u))
                                   : 0xFFFFu;
#pragma unroll
      for (int u = 0; u < kB; ++u) {
        if (c0 + 32 * u + lane < E) sq[c0 + 32 * u + lane] = (uint16_t)qq[u];
        if (fuse && qq[u] < nact) {  // (same bit formula as warp_panel_patterns)
          const uint32_t j = qq[u] >> tk_sh, lc = qq[u] & (tk - 1);
          const int r = ra[u], bit = ((r & 15) << 2) | (int)(lc & 3);
          atomicOr(&pat32[2 * (j * (nbk + 1) + (lc >> 2) * nbrow + (r >> 4)) + (bit >> 5)], 1u << (bit & 31));
        }
      }
    }
    w.patterns_done = fuse;
  } else {
    // merge ranking (as k_count): the rows are sorted runs of (column, entry) keys; ceil(log2(rows)) levels of
    // pairwise run merges, each key placed by one binary search in its partner run, ping-ponging with the
    // (now dead) staged columns; then first occurrences are counted. Row starts go to sq[256..] (E <= 256).
    static_assert(kWSortCap == 256 && kWSortCap * 8 <= 4 * (kWCap / 2 + 8), "merge buffer in the stage window");
    uint64_t* src = keys;
    uint64_t* dst = reinterpret_cast<uint64_t*>(my + L.off_stage);
    uint16_t* rs = sq + kWSortCap;
    const int nrows = w.nrows;
#pragma unroll
    for (int k = 0; k < (tm + 31) / 32; ++k) {
      const int r = lane + 32 * k;
      if (r < nrows) rs[r] = (uint16_t)(r == 0 ? 0u : w.st[k]);
    }
    if (lane == 0) rs[nrows] = (uint16_t)E;
    int levels = 0;
    while ((1 << levels) < nrows) ++levels;
    if (levels & 1) {  // the last level must land in `keys` (the values are staged into the window next)
      for (int i = lane; i < E; i += 32) dst[i] = src[i];
      uint64_t* t2 = src; src = dst; dst = t2;
    }
    __syncwarp();
    for (int l = 0; l < levels; ++l) {
      for (int x = lane; x < E; x += 32) {
        const uint64_t key = src[x];
        if ((uint32_t)key >= (uint32_t)E) continue;  // (stale slot: only after an unsorted row)
        const int r = srow[(uint32_t)key];
        const int g0 = (r >> (l + 1)) << (l + 1);
        const int gm = min(g0 + (1 << l), nrows), g1 = min(g0 + (2 << l), nrows);
        const int a0 = rs[g0], am = rs[gm], a1 = rs[g1];
        const bool left = r < gm;
        int lo = left ? am : a0, hi = left ? a1 : am;
        const int base = lo;
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (src[mid] < key) lo = mid + 1; else hi = mid;
        }
        const int pos = a0 + (left ? x - a0 : x - am) + (lo - base);
        if ((unsigned)pos < (unsigned)E) dst[pos] = key;  // (always, for sorted rows)
      }
      __syncwarp();
      uint64_t* t2 = src; src = dst; dst = t2;
    }
    for (int i = lane; i < E; i += 32) sq[i] = 0xFFFFu;  // (an unsorted row may leave entries unranked)
    __syncwarp();
    const int per = (E + 31) / 32, beg = lane * per;
    uint32_t sum = 0;
    for (int i = beg; i < beg + per && i < E; ++i)
      if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ++sum;
    uint32_t run = warp_excl_scan(sum, &nact);
    for (int i = beg; i < beg + per && i < E; ++i) {
      if (i == 0 || (keys[i] >> 32) != (keys[i - 1] >> 32)) ++run;
      if ((uint32_t)keys[i] < (uint32_t)E) sq[(uint32_t)keys[i]] = (uint16_t)(run - 1);
    }
    __syncwarp();
  }
  w.nact = nact;
  w.nblk = (nact + tk - 1) / tk;
  return true;
}

// Brick patterns (P:L132 fill_brick_nnz_pattern; bit = (r % 16) * 4 + q % 4, R3) of blocks [jb0, jb0 + nb) of a
// ranked warp-path panel into the warp's slot array (slot = (j - jb0) * (nbk + 1) + brick column * nbrow + brick
// row; one pad slot per block).
template <int tm, int tk>
__device__ __forceinline__ void warp_panel_patterns(const WarpPanel& w, uint8_t* my, const WarpLayout& L,
                                                    uint32_t jb0, uint32_t nb) {
  const int lane = threadIdx.x & 31;
  const uint8_t* srow = my + L.off_row;
  const uint16_t* sq = reinterpret_cast<const uint16_t*>(my + L.off_q);
  uint32_t* pat32 = reinterpret_cast<uint32_t*>(my + L.off_pat);
  constexpr int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  constexpr int tk_sh = tk == 16 ? 4 : 5;
  __syncwarp();  // every lane is done reading the previous chunk's patterns
  for (int i = lane; i < 2 * (int)nb * (nbk + 1); i += 32) pat32[i] = 0u;
  __syncwarp();
  const uint32_t q0 = jb0 * tk, q1 = min((jb0 + nb) * tk, w.nact);
  for (int c0 = 0; c0 < w.E; c0 += 32 * kB) {
    uint32_t qa[kB];
    int ra[kB];
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const int i = c0 + 32 * u + lane;
      qa[u] = i < w.E ? sq[i] : 0xFFFFFFFFu;
      ra[u] = i < w.E ? srow[i] : 0;
    }
#pragma unroll
    for (int u = 0; u < kB; ++u) {
      const uint32_t qq = qa[u];
      if (qq >= q0 && qq < q1) {
        const int r = ra[u];
        const uint32_t j = (qq >> tk_sh) - jb0, lc = qq & (tk - 1);
        const int bit = ((r & 15) << 2) | (int)(lc & 3);
        atomicOr(&pat32[2 * (j * (nbk + 1) + (lc >> 2) * nbrow + (r >> 4)) + (bit >> 5)], 1u << (bit & 31));
      }
    }
  }
  __syncwarp();
}

// Classification pre-pass: panels the warp path cannot take (more than kWCap entries, column span wider than
// the bitmap) are flagged and listed: those with more than kSmallCap entries (hubs) for the hub count kernel
// (panels above huge_cap, if > 0, from the end of biglist: that kernel claims them first), the others for the CTA
// count kernel. The two count kernels then share no input and run concurrently, before k_wbuild.
template <int tm, int tk>
__global__ void __launch_bounds__(32 * kWWarps) k_wclassify(const int64_t* __restrict__ rp,
                                                           const int32_t* __restrict__ ci, int64_t M, int64_t nnz,
                                                           int64_t P, uint8_t* __restrict__ listed,
                                                           uint32_t* __restrict__ list,
                                                           uint32_t* __restrict__ nlist,
                                                           uint32_t* __restrict__ biglist,
                                                           uint32_t* __restrict__ nbig,
                                                           uint32_t* __restrict__ nhuge, int64_t huge_cap) {
  pdl_wait();
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int64_t p = (int64_t)blockIdx.x * kWWarps + wid; p < P; p += (int64_t)gridDim.x * kWWarps) {
    WarpPanel w;
    // panels with <= kWSortCap entries take the warp path whatever their span (bitmap or merge ranking, decided
    // again in k_wbuild): no column reads for them
    bool ok = warp_panel_rows<tm, tk>(rp, M, nnz, p, w, nullptr);
    if (ok && w.E > kWSortCap) ok = warp_panel_span<tm>(w, [&](uint32_t i) { return ci[w.e0 + i]; });
    if (lane == 0) {
      listed[p] = ok ? 0 : 1;
      if (!ok) {
        if (w.Eall > kSmallCap) {
          if (huge_cap > 0 && w.Eall > huge_cap) biglist[P - atomicAdd(nhuge, 1u)] = (uint32_t)p;
          else biglist[atomicAdd(nbig, 1u)] = (uint32_t)p;
        } else {
          list[atomicAdd(nlist, 1u)] = (uint32_t)p;
        }
      }
    }
  }
}

// Decoupled look-back over panels (single-pass exclusive scan, warp granularity): st[p] holds the panel's
// aggregate (flag A) as soon as it is known, later its inclusive prefix (flag P). Panels are claimed in order
// through a ticket, so every predecessor belongs to a warp that is running or done.
#ifndef HRPB_LB_SLEEP
#define HRPB_LB_SLEEP 64
#endif
#ifndef HRPB_LB_WIN
#define HRPB_LB_WIN 1
#endif
constexpr int kLbWin = HRPB_LB_WIN;  // look-back windows of 32 states loaded per round (2, 4, 8: fewer rounds
                                     // -- 4.7 -> 2.1 per panel at 4 -- but measured slower builds)
#define kLbA (1ull << 62)
#define kLbP (2ull << 62)
#define kLbMask ((1ull << 62) - 1)
__device__ __forceinline__ uint64_t ld_relaxed_gpu(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_gpu(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
// One look-back over a state word carrying (blocks << 34 | bytes) (host checks both fit: blocks < 2^28,
// bytes < 2^34). Returns the exclusive prefix of the packed pair (the fields never carry into each other).
// Publishes the panel's aggregate (flag A; panel 0: its inclusive prefix, flag P). Work placed between this and
// warp_lb_wait gives the successors slack: they stall only until the aggregate is out, not until our wait ends.
__device__ __forceinline__ void warp_lb_publish(uint64_t* st, int64_t p, uint64_t agg) {
  if ((threadIdx.x & 31) == 0) st_relaxed_gpu(st + p, (p == 0 ? kLbP : kLbA) | agg);
}
#ifdef HRPB_BTRACE
__device__ unsigned long long g_lbstat[4];  // look-back: panels, load rounds, polls of unpublished states
#endif
__device__ __forceinline__ uint64_t warp_lb_wait(uint64_t* st, int64_t p, uint64_t agg) {
  const int lane = threadIdx.x & 31;
#ifdef HRPB_BTRACE
  unsigned rounds = 0, polls = 0;
#endif
  if (p == 0) {
    __syncwarp();
    return 0;
  }
  // The nearest inclusive prefix is typically ~150 panels back on c2a (its owners are still in their own
  // look-back); each round loads kLbWin windows of 32 states at once and walks them in order.
  uint64_t excl = 0;
  int64_t j = p - 1;
  bool done = false;
  while (!done) {
    uint64_t vw[kLbWin];
#pragma unroll
    for (int u = 0; u < kLbWin; ++u) {
      const int64_t idx = j - 32 * u - lane;
      vw[u] = idx >= 0 ? ld_relaxed_gpu(st + idx) : kLbP;
    }
#ifdef HRPB_BTRACE
    ++rounds;
#endif
#pragma unroll
    for (int u = 0; u < kLbWin; ++u) {
      const int64_t idx = j - 32 * u - lane;
      uint64_t v = vw[u];
      uint32_t pm;
      while (true) {  // only the states up to the nearest inclusive prefix are needed: wait for those alone
        pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const uint32_t zm = __ballot_sync(0xffffffffu, (v >> 62) == 0);
        const uint32_t need = pm ? ((pm & (0u - pm)) - 1u) : 0xFFFFFFFFu;  // lanes before the first P
        if (!(zm & need)) break;
        __nanosleep(HRPB_LB_SLEEP);  // back off: a spinning warp takes issue slots from the warps it waits for
#ifdef HRPB_BTRACE
        ++polls;
#endif
        if ((v >> 62) == 0) v = ld_relaxed_gpu(st + idx);
      }
      const int last = pm ? __ffs(pm) - 1 : 31;  // lanes 0..last contribute (lane `last` has the prefix)
      uint64_t x = lane <= last ? (v & kLbMask) : 0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      excl += x;
      if (pm) { done = true; break; }
    }
    j -= 32 * kLbWin;
  }
  if (lane == 0) st_relaxed_gpu(st + p, kLbP | (excl + agg));
#ifdef HRPB_BTRACE
  if (lane == 0) { atomicAdd(&g_lbstat[0], 1ull); atomicAdd(&g_lbstat[1], rounds); atomicAdd(&g_lbstat[2], polls); }
#endif
  __syncwarp();
  return excl;
}

// One block's HRPB-v1 metadata at blk (16-B aligned): header bytes colPtr[0..nbc] (stored bricks before each
// brick column), rows[nbr] (brick row of each stored brick), zero pad to 8 B -- assembled 8 bytes at a time --
// then the non-zero brick patterns in CSC slot order, and the zero tail padding after the nz values (R7).
template <int nbc, int nbrow>
__device__ __forceinline__ void emit_block_meta(uint8_t* blkp, const unsigned long long* pj, uint32_t nbr,
                                                uint32_t nz, uint32_t size) {
  constexpr int nbk = nbc * nbrow;
  uint64_t* blk = reinterpret_cast<uint64_t*>(blkp);
  const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
  uint64_t acc = 0;
  uint32_t nb = 1, k = 0, wi = 0;  // byte 0 = colPtr[0] = 0
#pragma unroll
  for (int bc = 0; bc < nbc; ++bc) {
#pragma unroll
    for (int br = 0; br < nbrow; ++br) k += pj[bc * nbrow + br] != 0ull;
    acc |= (uint64_t)k << (8 * (nb & 7));
    if ((++nb & 7) == 0) { blk[wi++] = acc; acc = 0; }
  }
  for (int bc = 0; bc < nbc; ++bc)
    for (int br = 0; br < nbrow; ++br) {
      const uint64_t v = pj[bc * nbrow + br];
      if (!v) continue;
      acc |= (uint64_t)br << (8 * (nb & 7));
      if ((++nb & 7) == 0) { blk[wi++] = acc; acc = 0; }
    }
  if (nb & 7) blk[wi++] = acc;
  for (int i = 0; i < nbk; ++i) {
    const uint64_t v = pj[i];
    if (v) blk[wi++] = v;
  }
  uint32_t* tail = reinterpret_cast<uint32_t*>(blkp + hdr + 8 * nbr + 4 * nz);
  for (uint32_t t = hdr + 8 * nbr + 4 * nz; t < size; t += 4) *tail++ = 0u;
}

// emit_block_meta with run-time brick shape (listed panels: one kernel for every TM / TK)
__device__ __forceinline__ void emit_block_meta_dyn(uint8_t* blkp, const unsigned long long* pj, int nbc, int nbrow,
                                                    uint32_t nbr, uint32_t nz, uint32_t size) {
  uint64_t* blk = reinterpret_cast<uint64_t*>(blkp);
  const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
  uint64_t acc = 0;
  uint32_t nb = 1, k = 0, wi = 0;  // byte 0 = colPtr[0] = 0
  for (int bc = 0; bc < nbc; ++bc) {
    for (int br = 0; br < nbrow; ++br) k += pj[bc * nbrow + br] != 0ull;
    acc |= (uint64_t)k << (8 * (nb & 7));
    if ((++nb & 7) == 0) { blk[wi++] = acc; acc = 0; }
  }
  for (int bc = 0; bc < nbc; ++bc)
    for (int br = 0; br < nbrow; ++br) {
      if (!pj[bc * nbrow + br]) continue;
      acc |= (uint64_t)br << (8 * (nb & 7));
      if ((++nb & 7) == 0) { blk[wi++] = acc; acc = 0; }
    }
  if (nb & 7) blk[wi++] = acc;
  for (int i = 0; i < nbc * nbrow; ++i) {
    const uint64_t v = pj[i];
    if (v) blk[wi++] = v;
  }
  uint32_t* tail = reinterpret_cast<uint32_t*>(blkp + hdr + 8 * nbr + 4 * nz);
  for (uint32_t t = hdr + 8 * nbr + 4 * nz; t < size; t += 4) *tail++ = 0u;
}

#ifdef HRPB_BTRACE
__device__ unsigned long long g_btrace[8];  // per-phase cycles summed over warps (diagnostic builds only)
#define BT_MARK(k) do { const long long t_ = clock64(); bt[k] += t_ - bt_last; bt_last = t_; } while (0)
#else
#define BT_MARK(k) do { } while (0)
#endif

// Fused pass for all panels: warp-path panels are ranked, their (blocks, bytes) published, the exclusive
// prefixes (blockedRowPtr, B2; panel byte offset, B4) found by look-back, and the panel emitted:
// sizePtr, HRPB-v1 headers + patterns + zero padding (R7), values in brick-CSC order at popcount
// ranks, activeCols with sentinel K (R2, R6). Listed panels only take part in the scan
// with the (nblk, bytes) their CTA / hub count produced; k_emit writes them afterwards.
// MODE 0: single pass (the look-back above). MODE 1 (count): every panel's packed (blocks << 34 | bytes) into
// lb[p], no emission; a device scan then gives the exclusive prefixes; MODE 2 (emit): the panel is ranked again and
// emitted at the scanned offset lb[p], no waiting. The look-back ties every warp to the slowest panel among the
// ~4K in flight (each waits for all predecessors' aggregates): on irregular matrices (c3: 4 us to 20 us panels)
// counting twice is cheaper than waiting.
template <int tm, int tk, int MODE>
__global__ void __launch_bounds__(32 * kWWarps, HRPB_WB_MINB) k_wbuild(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                        const float* __restrict__ vals, int64_t M, int64_t K,
                                                        int64_t nnz, int64_t P, const uint8_t* __restrict__ listed,
                                                        const uint32_t* __restrict__ nblk_listed,
                                                        const uint32_t* __restrict__ pbytes_listed,
                                                        uint32_t* __restrict__ ticket, uint64_t* __restrict__ lb,
                                                        uint32_t* __restrict__ brp,
                                                        uint64_t* __restrict__ poff, uint32_t* __restrict__ ac,
                                                        uint64_t* __restrict__ sp, uint8_t* __restrict__ packed,
                                                        uint32_t* status) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t dsm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WarpLayout L = warp_layout(tm, tk);
  uint8_t* my = dsm + (size_t)wid * L.bytes;
  constexpr int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  constexpr int kbs = nbk + 1;  // slot stride of a block: the +1 skews blocks across banks (the per-lane block
                                // loops and the pattern atomics hit one bank 16-way with a stride of nbk)
  const uint8_t* srow = my + L.off_row;
  const uint16_t* sq = reinterpret_cast<const uint16_t*>(my + L.off_q);
  const unsigned long long* pat = reinterpret_cast<const unsigned long long*>(my + L.off_pat);
  constexpr int tk_sh = tk == 16 ? 4 : 5;
  uint16_t* soff = reinterpret_cast<uint16_t*>(my + L.off_soff);
  uint64_t* vbase = reinterpret_cast<uint64_t*>(my + L.off_vbase);
  // 16-B cp.async staging needs 16-B aligned col_idx / values arrays
  const bool al16 = ((reinterpret_cast<uintptr_t>(ci) | reinterpret_cast<uintptr_t>(vals)) & 15) == 0;
#ifdef HRPB_BTRACE
  long long bt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, bt_last = clock64();
#endif
  while (true) {
    uint32_t t = 0;
    if (lane == 0) t = atomicAdd(ticket, 1u);
    const int64_t p = (int64_t)__shfl_sync(0xffffffffu, t, 0);
    BT_MARK(0);
    if (p >= P) break;
    WarpPanel w;
    w.E = 0;
    w.nblk = 0;
    uint32_t bytes = 0;
    int vsh = 0;
    constexpr uint32_t kChunkBlk = wslots(tm, tk) / nbk;  // blocks whose patterns fit the slot array
    static_assert(kChunkBlk <= 16, "prepared emission: lane j holds block j, codes carry j in 4 bits");
    // Prepared emission (bitmap-ranked panels whose blocks fit one pattern chunk, the common case): block sizes,
    // in-panel offsets, brick value offsets and every entry's destination are computed between publishing the
    // aggregate and waiting for the predecessors; after the look-back only the stores remain.
    bool prep = false;
    uint32_t pnbr = 0, pnz = 0, psize = 0, proff = 0;  // lane j: block j (prepared emission)
    const bool is_listed = listed[p] != 0;
    if (is_listed) {
      w.nblk = nblk_listed[p];
      bytes = pbytes_listed[p];
    } else {
      warp_panel_rows<tm, tk>(rp, M, nnz, p, w, status);  // (true: the classification pass agreed)
      BT_MARK(1);
      if (w.E > 0) {
        const int sh = warp_stage(ci, nnz, w.e0, w.E, my + L.off_stage, al16);
        warp_stage_wait();
        BT_MARK(2);
        const int32_t* scol = reinterpret_cast<const int32_t*>(my + L.off_stage) + sh;
        warp_panel_span<tm>(w, [&](uint32_t i) { return scol[i]; });
        warp_panel_rank<tm, tk>(scol, K, w, my, L, status);
        BT_MARK(3);
        __syncwarp();  // the staged columns are dead: the values go into the same window, landing meanwhile
        if (MODE != 1) vsh = warp_stage(vals, nnz, w.e0, w.E, my + L.off_stage, al16);
        prep = MODE != 1 && !w.sorted && w.nblk <= kChunkBlk;
        for (uint32_t jb0 = 0; jb0 < w.nblk; jb0 += kChunkBlk) {
          const uint32_t nb = min(kChunkBlk, w.nblk - jb0);
          if (!w.patterns_done) warp_panel_patterns<tm, tk>(w, my, L, jb0, nb);
          else __syncwarp();
          if (prep) break;
          for (uint32_t j = lane; j < nb; j += 32) {
            uint32_t nbr = 0, nz = 0;
#pragma unroll
            for (int i = 0; i < nbk; ++i) { const uint64_t v = pat[j * kbs + i]; nbr += v != 0ull; nz += __popcll(v); }
            bytes += block_bytes(nbc, nbr, nz);
          }
        }
        if (prep) {
          if ((uint32_t)lane < w.nblk) {
#pragma unroll
            for (int i = 0; i < nbk; ++i) {
              const uint64_t v = pat[lane * kbs + i];
              soff[lane * kbs + i] = (uint16_t)pnz;  // values of the earlier bricks of the block (CSC slot order)
              pnbr += v != 0ull;
              pnz += __popcll(v);
            }
            psize = block_bytes(nbc, pnbr, pnz);
          }
          proff = warp_excl_scan(psize, &bytes);
          if ((uint32_t)lane < w.nblk) vbase[lane] = proff + ((nbc + 1 + pnbr + 7) & ~7u) + 8 * pnbr;  // relative
        } else {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
        }
      }
    }
    BT_MARK(4);
    const uint64_t agg = ((uint64_t)w.nblk << 34) | bytes;
    if (MODE == 1) {  // count pass: the aggregate only (the device scan turns lb into exclusive prefixes)
      if (lane == 0) lb[p] = agg;
      continue;
    }
    if (MODE == 0) warp_lb_publish(lb, p, agg);
    if (prep) {  // entry destinations: sq[i] <- (block << 11) | value index in the block (0xFFFF stays invalid)
      __syncwarp();
      uint16_t* sqw = reinterpret_cast<uint16_t*>(my + L.off_q);
      for (int c0 = 0; c0 < w.E; c0 += 32 * kB) {
        uint32_t qa[kB], code[kB];
        int ra[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int i = c0 + 32 * u + lane;
          qa[u] = i < w.E ? sq[i] : 0xFFFFu;
          ra[u] = i < w.E ? srow[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          code[u] = 0xFFFFu;
          if (qa[u] < w.nact) {
            const int r = ra[u];
            const uint32_t j = qa[u] >> tk_sh, lc = qa[u] & (tk - 1);
            const int bit = ((r & 15) << 2) | (int)(lc & 3);
            const uint32_t slot = j * kbs + (lc >> 2) * nbrow + (r >> 4);
            code[u] = (j << 11) | (soff[slot] + __popcll(pat[slot] & ((1ull << bit) - 1ull)));
          }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u)
          if (c0 + 32 * u + lane < w.E) sqw[c0 + 32 * u + lane] = (uint16_t)code[u];
      }
    }
    const uint64_t ex = MODE == 0 ? warp_lb_wait(lb, p, agg) : lb[p];
    BT_MARK(5);
    const uint32_t b0 = (uint32_t)(ex >> 34);
    const uint64_t pbase = ex & ((1ull << 34) - 1);
    if (lane == 0) {
      brp[p] = b0;
      poff[p] = pbase;
      if (p == P - 1) { brp[P] = b0 + w.nblk; poff[P] = pbase + bytes; }
    }
    if (is_listed || w.E == 0) continue;
    const uint32_t nblk = w.nblk;
    const int E = w.E;
    uint64_t carry = pbase;
    warp_stage_wait();
    const float* sval = reinterpret_cast<const float*>(my + L.off_stage) + vsh;
    for (int64_t t = w.nact + lane; t < (int64_t)nblk * tk; t += 32) ac[(int64_t)b0 * tk + t] = (uint32_t)K;
    // activeCols (R6, R23): the panel's distinct columns in ascending order, from the ranking structures
    uint32_t* acp = ac + (int64_t)b0 * tk;
    if (!w.sorted) {
      // a non-zero bitmap word at a time, its 32 bits across the lanes: lane l writes bit l's column at its rank
      const uint32_t* bm = reinterpret_cast<const uint32_t*>(my);
      const uint32_t* pre = reinterpret_cast<const uint32_t*>(my + L.off_pre);
      for (int k = 0; k < (w.nbw + 31) / 32; ++k) {
        const uint32_t mine = 32 * k + lane < w.nbw ? bm[32 * k + lane] : 0u;
        uint32_t nzw = __ballot_sync(0xffffffffu, mine != 0u);
        while (nzw) {
          const int kk = __ffs(nzw) - 1;
          nzw &= nzw - 1;
          const int wd = 32 * k + kk;
          const uint32_t bits = __shfl_sync(0xffffffffu, mine, kk);
          if ((bits >> lane) & 1u) acp[pre[wd] + __popc(bits & ((1u << lane) - 1u))] = (uint32_t)(w.mn + 32 * wd + lane);
        }
      }
    } else {
      const uint64_t* keys = reinterpret_cast<const uint64_t*>(my);
      for (int i = lane; i < w.E; i += 32) {
        const uint32_t e = (uint32_t)keys[i];
        if (e < (uint32_t)w.E && sq[e] < w.nact) acp[sq[e]] = (uint32_t)(keys[i] >> 32);  // (guards: invalid CSR)
      }
    }
    if (prep) {
      if ((uint32_t)lane < nblk) {
        const uint64_t off = pbase + proff;
        sp[b0 + lane] = off;
        emit_block_meta<nbc, nbrow>(packed + off, pat + lane * kbs, pnbr, pnz, psize);
      }
      for (int c0 = 0; c0 < E; c0 += 32 * kB) {  // values at the prepared destinations (loads of the round first)
        uint32_t ca[kB];
        float va[kB];
        uint64_t ba[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int i = c0 + 32 * u + lane;
          ca[u] = i < E ? sq[i] : 0xFFFFu;
          va[u] = i < E ? sval[i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) ba[u] = ca[u] != 0xFFFFu ? vbase[ca[u] >> 11] : 0ull;
#pragma unroll
        for (int u = 0; u < kB; ++u)
          if (ca[u] != 0xFFFFu) reinterpret_cast<float*>(packed + pbase + ba[u])[ca[u] & 0x7FFu] = va[u];
      }
      BT_MARK(6);
      continue;
    }
    for (uint32_t jb0 = 0; jb0 < nblk; jb0 += kChunkBlk) {
      const uint32_t nbch = min(kChunkBlk, nblk - jb0);
      if (jb0 > 0) warp_panel_patterns<tm, tk>(w, my, L, jb0, nbch);  // (chunk 0 is still in place if alone)
      else if (nblk > kChunkBlk) warp_panel_patterns<tm, tk>(w, my, L, 0, nbch);
      for (uint32_t c0 = 0; c0 < nbch; c0 += 32) {  // blocks: sizes, in-panel scan, headers, patterns, padding
        const uint32_t j = c0 + lane;  // block jb0 + j of the panel
        uint32_t nbr = 0, nz = 0, size = 0;
        if (j < nbch) {
#pragma unroll
          for (int i = 0; i < nbk; ++i) {
            const uint64_t v = pat[j * kbs + i];
            soff[j * kbs + i] = (uint16_t)nz;  // values of the earlier bricks of the block (CSC slot order)
            nbr += v != 0ull;
            nz += __popcll(v);
          }
          size = block_bytes(nbc, nbr, nz);
        }
        uint32_t tot;
        const uint64_t off = carry + warp_excl_scan(size, &tot);
        if (j < nbch) {
          sp[b0 + jb0 + j] = off;
          emit_block_meta<nbc, nbrow>(packed + off, pat + j * kbs, nbr, nz, size);
          vbase[j] = off + ((nbc + 1 + nbr + 7) & ~7u) + 8 * nbr;
        }
        carry += tot;
      }
      __syncwarp();
      const uint32_t q0 = jb0 * tk, q1 = min((jb0 + nbch) * tk, w.nact);
      for (int c0 = 0; c0 < E; c0 += 32 * kB) {  // values of this chunk's blocks (loads of the round first)
        uint32_t qa[kB], oa[kB];
        int ra[kB];
        float va[kB];
        uint64_t ba[kB];
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const int i = c0 + 32 * u + lane;
          qa[u] = i < E ? sq[i] : 0xFFFFFFFFu;
          ra[u] = i < E ? srow[i] : 0;
          va[u] = i < E ? sval[i] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kB; ++u) {
          const uint32_t qq = qa[u];
          if (qq >= q0 && qq < q1) {
            const int r = ra[u];
            const uint32_t j = (qq >> tk_sh) - jb0, lc = qq & (tk - 1);
            const int bit = ((r & 15) << 2) | (int)(lc & 3);
            const uint32_t slot = j * kbs + (lc >> 2) * nbrow + (r >> 4);
            oa[u] = soff[slot] + __popcll(pat[slot] & ((1ull << bit) - 1ull));
            ba[u] = vbase[j];
          }
        }
#pragma unroll
        for (int u = 0; u < kB; ++u)
          if (qa[u] >= q0 && qa[u] < q1) reinterpret_cast<float*>(packed + ba[u])[oa[u]] = va[u];
      }
      __syncwarp();
    }
    BT_MARK(6);
  }
#ifdef HRPB_BTRACE
  if (lane == 0)
    for (int k = 0; k < 7; ++k) atomicAdd(&g_btrace[k], (unsigned long long)bt[k]);
#endif
}

// ------------------------------------------------------------------ pass A (CTA), listed panels with <= kSmallCap entries
// One CTA per listed panel, claimed dynamically ("for row_panel in rowPanels_chunk"). q[e] = rank of
// col_idx[e] among the panel's distinct columns (ascending, R23; "active_cols = uniq(cols[...])"),
// nblk = ceil(nact/TK) (R1), brick patterns (bit = (r % 16) * 4 + q % 4, R3) and the panel's total block bytes.
// Ranking, by the panel's column layout:
//  * windowed byte maps (clustered columns, e.g. FEM stencils, banded panels too wide for the warp path): the
//    1024-column windows the panel touches are found from its row "breaks" only (the entries starting a row or a
//    new window within a row: rows are sorted) through a window-occupancy bitmap over all K/1024 windows, whose
//    popcount prefix gives each window its ordinal; each entry then marks a byte in its window's 1-KB byte map
//    (plain stores: no same-word atomics), the byte maps become bitmap words, and rank = word prefix + popc;
//  * more than kMaxWin windows (scattered columns, e.g. R-MAT) or K > 32M: a CTA radix sort (CUB) of the
//    (column, entry) pairs, rank = number of distinct columns before the entry's in sorted order.
constexpr int kMidThreads = 256;
constexpr int kMidItems = kSmallCap / kMidThreads;  // 8 entries per thread in the sort path
constexpr int kWinBits = 10;                        // window = 1024 columns = 32 bitmap words
constexpr int kMaxWin = 16;                         // windows per panel on the windowed path
constexpr int kOccWords = 1024;                     // window-occupancy words: K <= 2^(15 + kWinBits) = 32M
using MidSort = cub::BlockRadixSort<uint32_t, kMidThreads, kMidItems, uint32_t, 6>;  // <= 2048 entries
using MidSort2 = cub::BlockRadixSort<uint32_t, kMidThreads, 2, uint32_t, 6>;         // <= 512 entries
struct MidWin {
  uint8_t bmap[kMaxWin << kWinBits];  // byte map per window
  uint32_t bits[kMaxWin * 32];        // bitmap words
  uint32_t pre[kMaxWin * 32];         // exclusive popcount prefix per word
};
// two-level bitmap over the whole column space (K <= 32 * 32 * kWordOccWords): occ2 = one bit per 32-column word,
// the occupied words get dense ordinals (popcount prefix, u16: <= kSmallCap of them), mask[ordinal] = the word's
// column bits, mpre = exclusive popcount prefix over the masks; rank = mpre[ord] + popc(mask[ord] & lower bits)
constexpr int kWordOccWords = 4096;  // K <= 2^22
struct Mid2L {
  uint32_t occ2[kWordOccWords];
  uint16_t opre[kWordOccWords];
  uint32_t mask[kSmallCap];
  uint16_t mpre[kSmallCap];
};
union MidUnion {
  MidWin win;
  Mid2L two;
  typename MidSort::TempStorage sort;
  typename MidSort2::TempStorage sort2;
};
struct MidSmem {
  uint32_t col[kSmallCap];
  uint32_t q[kSmallCap];  // window ordinal, then rank
  uint8_t row[kSmallCap];
  uint32_t occ[kOccWords];
  uint32_t occpre[kOccWords];
  uint32_t last_key[kMidThreads];
  MidUnion u;
  // brick patterns follow (dynamic size: (kSmallCap / tk + 1) * nbk * 8 bytes)
};
__host__ __device__ constexpr size_t mid_smem_bytes(int tm, int tk) {
  return sizeof(MidSmem) + (size_t)(kSmallCap / tk + 1) * (tk / HRPB_BRICK_K) * (tm / HRPB_BRICK_M) * 8 + 16;
}

// rank of every entry among the distinct columns: radix sort of (column, entry), head flags, CTA scan
template <typename SortT, int ITEMS>
__device__ __forceinline__ uint32_t mid_sort_rank(MidSmem& S, typename SortT::TempStorage& tmp, int E, int kb,
                                                  uint32_t* s_scan) {
  const int tid = threadIdx.x;
  uint32_t key[ITEMS], val[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const int i = tid * ITEMS + k;
    key[k] = i < E ? S.col[i] : 0xFFFFFFFFu;
    val[k] = (uint32_t)i;
  }
  SortT(tmp).Sort(key, val, 0, kb);
  S.last_key[tid] = key[ITEMS - 1];
  __syncthreads();
  uint32_t heads = 0, nact = 0;
  uint32_t prev = tid ? S.last_key[tid - 1] : 0xFFFFFFFFu;
  bool hd[ITEMS];
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    const bool valid = val[k] < (uint32_t)E;
    hd[k] = valid && (tid * ITEMS + k == 0 || key[k] != prev);
    heads += hd[k];
    prev = key[k];
  }
  uint32_t run = block_excl_scan<kMidThreads>(heads, &nact, s_scan);
#pragma unroll
  for (int k = 0; k < ITEMS; ++k) {
    run += hd[k];
    if (val[k] < (uint32_t)E) S.q[val[k]] = run - 1;
  }
  return nact;
}

#ifndef HRPB_COUNT_MINB
#define HRPB_COUNT_MINB 3  // 80 registers: 3 CTAs per SM (shared memory allows 3; c3 1.86 -> 1.52 ms, c5 0.79 -> 0.57 ms)
#endif
__global__ void __launch_bounds__(kMidThreads, HRPB_COUNT_MINB) k_count(const int64_t* __restrict__ rp,
                                                      const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                      int64_t nnz, int tm, int tk, uint32_t* __restrict__ q,
                                                      uint32_t* __restrict__ nact_out,
                                                      uint32_t* __restrict__ nblk_out,
                                                      uint32_t* __restrict__ pbytes_out,
                                                      uint64_t* __restrict__ gpat,
                                                      const uint32_t* __restrict__ midlist,
                                                      const uint32_t* __restrict__ nmid,
                                                      uint32_t* __restrict__ biglist,
                                                      uint32_t* __restrict__ nbig, uint32_t* work, uint32_t* status,
                                                      uint32_t* __restrict__ nhuge, int64_t huge_cap, int64_t P) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t dsm[];
  MidSmem& S = *reinterpret_cast<MidSmem*>(dsm);
  unsigned long long* s_pat = reinterpret_cast<unsigned long long*>(dsm + ((sizeof(MidSmem) + 15) & ~(size_t)15));
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_scan[kMidThreads / 32 + 1];
  __shared__ uint32_t s_t;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t count = *nmid;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const int occ_words = (int)min((int64_t)kOccWords, ceil_div(ceil_div(K, 1 << kWinBits), 32));
  const bool occ_ok = ceil_div(K, 1 << kWinBits) <= 32 * kOccWords;
  int kb = 1;
  while (kb < 32 && (1ll << kb) < K) ++kb;  // sort bits: columns < K <= 2^kb
  while (true) {
    if (tid == 0) s_t = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t t = s_t;
    if (t >= count) break;
    const int64_t p = midlist[t];
    load_panel_rows(rp, M, nnz, tm, p, s_rp, status);  // (barriers: also orders s_t's read)
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = s_rp[0];
    const int E = (int)min((int64_t)kSmallCap + 1, s_rp[nrows] - e0);
    if (E > kSmallCap) {  // CTA-uniform: handled by the hub kernel
      // (huge_cap > 0: panels above it are listed from the end of biglist, so the hub kernel claims them first)
      if (tid == 0) {
        if (huge_cap > 0 && s_rp[nrows] - e0 > huge_cap) biglist[P - atomicAdd(nhuge, 1u)] = (uint32_t)p;
        else biglist[atomicAdd(nbig, 1u)] = (uint32_t)p;
      }
      continue;
    }
    // entries -> shared memory (column clamped into [0, K) for memory safety; invalid CSR is flagged), row map
    bool bad_range = false;
    for (int i = tid; i < E; i += kMidThreads) {
      const int32_t c = ci[e0 + i];
      if (c < 0 || c >= K) bad_range = true;
      S.col[i] = (uint32_t)min(max(c, 0), (int32_t)(K - 1));
    }
    for (int i = tid; i < occ_words; i += kMidThreads) S.occ[i] = 0u;
    for (int r = warp; r < nrows; r += kMidThreads / 32) {
      const int b = (int)(s_rp[r] - e0), e = (int)(s_rp[r + 1] - e0);
      for (int i = b + lane; i < e; i += 32) S.row[i] = (uint8_t)r;
    }
    if (__any_sync(0xffffffffu, bad_range) && lane == 0) atomicOr(status, ST_COL_RANGE);
    __syncthreads();
    // in-row order and the window breaks: a row's first entry or its first entry in a new window
    bool bad_order = false;
    for (int i = tid; i < E; i += kMidThreads) {
      const uint32_t c = S.col[i];
      const bool same_row = i > 0 && S.row[i - 1] == S.row[i];
      if (same_row && S.col[i - 1] >= c) bad_order = true;
      if (occ_ok && (!same_row || (S.col[i - 1] >> kWinBits) != (c >> kWinBits))) {
        const uint32_t w = c >> kWinBits;
        atomicOr(&S.occ[w >> 5], 1u << (w & 31));
      }
    }
    if (__any_sync(0xffffffffu, bad_order) && lane == 0) atomicOr(status, ST_COL_ORDER);
    __syncthreads();
    uint32_t nwin = 0xFFFFFFFFu;
    if (occ_ok) {  // window ordinals: exclusive popcount prefix over the occupancy words (<= 4 per thread)
      uint32_t cnt[kOccWords / kMidThreads], sum = 0;
#pragma unroll
      for (int k = 0; k < kOccWords / kMidThreads; ++k) {
        const int wi = tid * (kOccWords / kMidThreads) + k;
        cnt[k] = wi < occ_words ? __popc(S.occ[wi]) : 0u;
        sum += cnt[k];
      }
      uint32_t run = block_excl_scan<kMidThreads>(sum, &nwin, s_scan);
#pragma unroll
      for (int k = 0; k < kOccWords / kMidThreads; ++k) {
        const int wi = tid * (kOccWords / kMidThreads) + k;
        if (wi < occ_words) S.occpre[wi] = run;
        run += cnt[k];
      }
    }
    uint32_t nact = 0;
    if (nwin <= (uint32_t)kMaxWin) {
      // ---- windowed byte maps
      uint32_t* bm32 = reinterpret_cast<uint32_t*>(S.u.win.bmap);
      for (int i = tid; i < (int)nwin << (kWinBits - 2); i += kMidThreads) bm32[i] = 0u;
      __syncthreads();  // (also publishes occpre)
      for (int i = tid; i < E; i += kMidThreads) {
        const uint32_t c = S.col[i], w = c >> kWinBits;
        const uint32_t k = S.occpre[w >> 5] + __popc(S.occ[w >> 5] & ((1u << (w & 31)) - 1u));
        S.q[i] = k;
        S.u.win.bmap[(k << kWinBits) | (c & ((1u << kWinBits) - 1u))] = 1;
      }
      __syncthreads();
      constexpr int kPer = kMaxWin * 32 / kMidThreads;  // bitmap words per thread
      uint32_t cnt[kPer], sum = 0;
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int wd = tid * kPer + k;
        uint32_t word = 0;
        if (wd < (int)nwin * 32) {
          const uint4* src = reinterpret_cast<const uint4*>(S.u.win.bmap + 32 * wd);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint4 v = src[h];
            const uint32_t x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int j = 0; j < 4; ++j)  // bytes are 0 / 1: bits 0, 8, 16, 24 -> a nibble
              word |= ((x[j] | (x[j] >> 7) | (x[j] >> 14) | (x[j] >> 21)) & 0xFu) << (16 * h + 4 * j);
          }
        }
        cnt[k] = __popc(word);
        sum += cnt[k];
        if (wd < (int)nwin * 32) S.u.win.bits[wd] = word;
      }
      uint32_t run = block_excl_scan<kMidThreads>(sum, &nact, s_scan);
#pragma unroll
      for (int k = 0; k < kPer; ++k) {
        const int wd = tid * kPer + k;
        if (wd < (int)nwin * 32) S.u.win.pre[wd] = run;
        run += cnt[k];
      }
      __syncthreads();
      for (int i = tid; i < E; i += kMidThreads) {
        const uint32_t c = S.col[i];
        const uint32_t wd = (S.q[i] << (kWinBits - 5)) | ((c >> 5) & ((1u << (kWinBits - 5)) - 1u));
        S.q[i] = S.u.win.pre[wd] + __popc(S.u.win.bits[wd] & ((1u << (c & 31)) - 1u));
      }
    } else if (K <= 32ll * 32 * kWordOccWords) {
      // ---- two-level bitmap (scattered columns, e.g. R-MAT): O(E + K / 1024) shared-memory work per panel
      Mid2L& T = S.u.two;
      __syncthreads();  // (occpre readers done before the union is reused)
      for (int i = tid; i < kWordOccWords / 4; i += kMidThreads) reinterpret_cast<uint4*>(T.occ2)[i] = make_uint4(0, 0, 0, 0);
      for (int i = tid; i < E; i += kMidThreads) T.mask[i] = 0u;
      __syncthreads();
      for (int i = tid; i < E; i += kMidThreads) {
        const uint32_t w = S.col[i] >> 5;
        atomicOr(&T.occ2[w >> 5], 1u << (w & 31));
      }
      __syncthreads();
      constexpr int kPer = kWordOccWords / kMidThreads;  // occupancy words per thread (16)
      {
        uint32_t cnt[kPer], sum = 0;
#pragma unroll
        for (int k = 0; k < kPer / 4; ++k) {
          const uint4 v = reinterpret_cast<const uint4*>(T.occ2)[tid * (kPer / 4) + k];
          cnt[4 * k] = __popc(v.x); cnt[4 * k + 1] = __popc(v.y); cnt[4 * k + 2] = __popc(v.z); cnt[4 * k + 3] = __popc(v.w);
        }
#pragma unroll
        for (int k = 0; k < kPer; ++k) sum += cnt[k];
        uint32_t nocc;
        uint32_t run = block_excl_scan<kMidThreads>(sum, &nocc, s_scan);
#pragma unroll
        for (int k = 0; k < kPer; k += 2) {
          reinterpret_cast<uint32_t*>(T.opre)[(tid * kPer + k) >> 1] = run | ((run + cnt[k]) << 16);
          run += cnt[k] + cnt[k + 1];
        }
      }
      __syncthreads();
      for (int i = tid; i < E; i += kMidThreads) {
        const uint32_t c = S.col[i], w = c >> 5;
        const uint32_t o = T.opre[w >> 5] + __popc(T.occ2[w >> 5] & ((1u << (w & 31)) - 1u));
        S.q[i] = o;
        atomicOr(&T.mask[o], 1u << (c & 31));
      }
      __syncthreads();
      {
        constexpr int kPerM = kSmallCap / kMidThreads;  // masks per thread (8)
        uint32_t cnt[kPerM], sum = 0;
#pragma unroll
        for (int k = 0; k < kPerM; ++k) {
          const int o = tid * kPerM + k;
          cnt[k] = o < E ? __popc(T.mask[o]) : 0u;
          sum += cnt[k];
        }
        uint32_t run = block_excl_scan<kMidThreads>(sum, &nact, s_scan);
#pragma unroll
        for (int k = 0; k < kPerM; ++k) {
          const int o = tid * kPerM + k;
          if (o < E) T.mpre[o] = (uint16_t)run;
          run += cnt[k];
        }
      }
      __syncthreads();
      for (int i = tid; i < E; i += kMidThreads) {
        const uint32_t c = S.col[i], o = S.q[i];
        S.q[i] = T.mpre[o] + __popc(T.mask[o] & ((1u << (c & 31)) - 1u));
      }
    } else {
      // ---- CTA radix sort of (column, entry); padding keys sort last (stable sort, entry >= E)
      __syncthreads();  // (occpre readers done before the union is reused)
      if (E <= 2 * kMidThreads) nact = mid_sort_rank<MidSort2, 2>(S, S.u.sort2, E, kb, s_scan);
      else nact = mid_sort_rank<MidSort, kMidItems>(S, S.u.sort, E, kb, s_scan);
    }
    // patterns (fill_brick_nnz_pattern): brick i = bc * (TM/16) + br in CSC order
    const uint32_t nblk = (nact + tk - 1) / tk;
    const int nbricks = (int)nblk * nbk;
    for (int i = tid; i < nbricks; i += kMidThreads) s_pat[i] = 0ull;
    __syncthreads();
    for (int i = tid; i < E; i += kMidThreads) {
      const uint32_t qq = S.q[i], r = S.row[i];
      q[e0 + i] = qq;
      const uint32_t j = qq / tk, lc = qq % tk;
      const int bit = (int)(((r & 15) << 2) | (lc & 3));
      // 32-bit OR on the half holding the bit (a 64-bit shared atomicOr is a CAS loop on sm_100)
      uint32_t* half = reinterpret_cast<uint32_t*>(&s_pat[j * nbk + (lc >> 2) * nbrow + (r >> 4)]) + (bit >> 5);
      atomicOr(half, 1u << (bit & 31));
    }
    __syncthreads();
    uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
    for (int i = tid; i < nbricks; i += kMidThreads) gp[i] = s_pat[i];
    uint32_t bytes = 0;
    for (uint32_t j = tid; j < nblk; j += kMidThreads) {
      uint32_t nbr = 0, nz = 0;
      for (int i = 0; i < nbk; ++i) { const uint64_t v = s_pat[j * nbk + i]; nbr += v != 0ull; nz += __popcll(v); }
      bytes += block_bytes(nbc, nbr, nz);
    }
    uint32_t total;
    block_excl_scan<kMidThreads>(bytes, &total, s_scan);  // (barriers: shared state is free for the next panel)
    if (tid == 0) { nact_out[p] = nact; nblk_out[p] = nblk; pbytes_out[p] = total; }
  }  // panel loop
}

// ------------------------------------------------------------------ pass A, panels with > kSmallCap entries
// Persistent CTAs over the hub-panel list. Ranks by a two-level bitmap over the column space: bm (one bit per
// column, W = K/32 words) and occ (one bit per bm word). Only the words a panel touches are visited: occupied
// words get dense ordinals (popcount prefix over occ), their popcounts are scanned densely, and
// rank(c) = dense prefix of c's word + popcount of the lower bits. The bitmaps are zero between panels (cleared
// word by word after use, zeroed once per CTA at its first panel), so the work is O(entries + K/1024) per panel
// instead of O(column span) (R-MAT panels span all 4M columns with a few thousand entries).
__global__ void __launch_bounds__(kBigThreads) k_count_big(const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                          int64_t nnz, int tm, int tk, uint32_t* __restrict__ q,
                                                          uint32_t* __restrict__ nact_out,
                                                          uint32_t* __restrict__ nblk_out,
                                                          uint32_t* __restrict__ pbytes_out,
                                                          uint64_t* __restrict__ gpat,
                                                          const uint32_t* __restrict__ biglist,
                                                          const uint32_t* __restrict__ nbig, uint32_t* scratch,
                                                          int64_t words_per_cta, uint32_t* work,
                                                          uint32_t* status) {
  pdl_wait();
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_scan[kBigThreads / 32 + 1];
  __shared__ uint32_t s_t;
  const int64_t W = words_per_cta;          // >= K/32 + 2
  const int64_t W1 = (W + 31) / 32;         // occupancy words
  uint32_t* bm = scratch + (int64_t)blockIdx.x * (2 * W + 2 * W1);
  uint32_t* dense = bm + W;                 // popcount prefix of the occupied words, in ordinal order
  uint32_t* occ = dense + W;
  uint32_t* occ_pre = occ + W1;
  const uint32_t count = *nbig;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  // hubs are claimed dynamically (sizes are power-law: a static round robin left CTAs 1.4x their mean share)
  bool zeroed = false;
  while (true) {
    if (threadIdx.x == 0) s_t = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t t = s_t;
    __syncthreads();
    if (t >= count) break;
    if (!zeroed) {  // establish the all-zero invariant at the CTA's first hub
      for (int64_t i = threadIdx.x; i < W; i += blockDim.x) bm[i] = 0u;
      for (int64_t i = threadIdx.x; i < W1; i += blockDim.x) occ[i] = 0u;
      __threadfence_block();
      zeroed = true;
    }
    const int64_t p = biglist[t];
    load_panel_rows(rp, M, nnz, tm, p, s_rp, status);  // (barriers: also orders the zeroing above)
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = s_rp[0], e1 = s_rp[nrows];
    // (1) bits + occupancy + validation
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int32_t c = ci[e];
      if (c < 0 || c >= K) { atomicOr(status, ST_COL_RANGE); continue; }
      const int r = row_of(s_rp, nrows, e);
      if (e > s_rp[r] && ci[e - 1] >= c) atomicOr(status, ST_COL_ORDER);
      const uint32_t w = (uint32_t)c >> 5;
      atomicOr(&bm[w], 1u << (c & 31));        // (results unused: fire-and-forget reductions, no round trip)
      atomicOr(&occ[w >> 5], 1u << (w & 31));
    }
    __threadfence_block();
    __syncthreads();
    // (2) ordinals of the occupied words: exclusive popcount prefix over occ (W1 words, per-thread runs)
    const int64_t per = (W1 + blockDim.x - 1) / blockDim.x;
    const int64_t beg = threadIdx.x * per, end = min(W1, beg + per);
    uint32_t sum = 0;
    for (int64_t i = beg; i < end; ++i) sum += __popc(__ldcg(&occ[i]));
    uint32_t nocc;
    uint32_t run = block_excl_scan<kBigThreads>(sum, &nocc, s_scan);
    for (int64_t i = beg; i < end; ++i) {
      occ_pre[i] = run;
      // (3) popcount of every occupied word at its ordinal, 8 loads in flight before their stores
      uint32_t o = __ldcg(&occ[i]), k = run;
      while (o) {
        uint32_t v[8];
        int n = 0;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          v[u] = 0u;
          if (o) {
            const int b = __ffs(o) - 1;
            o &= o - 1;
            v[u] = __ldcg(&bm[i * 32 + b]);
            n = u + 1;
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (u < n) dense[k + u] = __popc(v[u]);
        k += n;
      }
      run = k;
    }
    __threadfence_block();
    __syncthreads();
    // (4) dense exclusive scan of the occupied words' popcounts (in place, chunks of blockDim)
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < nocc; c0 += blockDim.x) {
      const uint32_t i = c0 + threadIdx.x;
      const uint32_t v = i < nocc ? __ldcg(&dense[i]) : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<kBigThreads>(v, &tot, s_scan);
      if (i < nocc) dense[i] = carry + ex;
      carry += tot;
    }
    const uint32_t nact = carry;
    const uint32_t nblk = (nact + tk - 1) / tk;
    unsigned long long* gp = reinterpret_cast<unsigned long long*>(gpat + pat_base(e0, p, nbk, tk));
    for (int64_t i = threadIdx.x; i < (int64_t)nblk * nbk; i += blockDim.x) gp[i] = 0ull;
    __threadfence_block();
    __syncthreads();
    // (5) ranks and patterns (fill_brick_nnz_pattern)
    constexpr int kU = 4;  // entries per thread per round, every load of the round before its stores
    for (int64_t eb = e0 + threadIdx.x; eb < e1; eb += (int64_t)kU * blockDim.x) {
      int32_t c[kU];
      uint32_t ord[kU], qq[kU], wb[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t e = eb + (int64_t)u * blockDim.x;
        c[u] = e < e1 ? ci[e] : -1;
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        ord[u] = 0u;
        wb[u] = 0u;
        if (c[u] >= 0 && c[u] < K) {
          const uint32_t w = (uint32_t)c[u] >> 5, w1 = w >> 5;
          ord[u] = __ldcg(&occ_pre[w1]) + __popc(__ldcg(&occ[w1]) & ((1u << (w & 31)) - 1u));
          wb[u] = __ldcg(&bm[w]);
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u)
        qq[u] = (c[u] >= 0 && c[u] < K) ? __ldcg(&dense[ord[u]]) + __popc(wb[u] & ((1u << (c[u] & 31)) - 1u))
                                         : 0xFFFFFFFFu;
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t e = eb + (int64_t)u * blockDim.x;
        if (e >= e1) continue;
        q[e] = qq[u];
        if (qq[u] == 0xFFFFFFFFu) continue;
        const int r = row_of(s_rp, nrows, e);
        const uint32_t j = qq[u] / tk, lc = qq[u] % tk;
        atomicOr(&gp[(int64_t)j * nbk + (lc >> 2) * nbrow + (r >> 4)], 1ull << (((r & 15) << 2) | (lc & 3)));
      }
    }
    __threadfence_block();
    __syncthreads();
    // (6) block sizes; clear the touched bitmap words and the occupancy words (invariant for the next panel)
    uint32_t bytes = 0;
    for (int64_t j = threadIdx.x; j < nblk; j += blockDim.x) {
      uint32_t nbr = 0, nz = 0;
      for (int i = 0; i < nbk; ++i) {
        const unsigned long long v = __ldcg(&gp[j * nbk + i]);
        nbr += v != 0ull;
        nz += __popcll(v);
      }
      bytes += block_bytes(nbc, nbr, nz);
    }
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int32_t c = ci[e];
      if (c >= 0 && c < K) bm[(uint32_t)c >> 5] = 0u;
    }
    for (int64_t i = beg; i < end; ++i) occ[i] = 0u;
    uint32_t total;
    block_excl_scan<kBigThreads>(bytes, &total, s_scan);  // (barriers: the clears are done before the next panel)
    if (threadIdx.x == 0) { nact_out[p] = nact; nblk_out[p] = nblk; pbytes_out[p] = total; }
    __threadfence_block();
  }
}

// ------------------------------------------------------------------ hub panels (> kSmallCap entries), dense passes
// One CTA per hub panel (claimed dynamically, power-law sizes). The column space is walked in passes of
// kHubPassCols columns with a dense bitmap in shared memory: set the bits of the pass's entries (per-row entry
// ranges of each pass come from one boundary sweep: rows are sorted), popcount prefix per 32-word group (u32) and
// per word within its group (u16), rank = prefix + popc(lower bits) (R23: ascending distinct columns). Ranks go to
// q[e]; the ranks of a pass are one contiguous range, so its blocks' brick patterns are built in a shared-memory
// window (shared atomics) and flushed to global memory once complete (a pass's last, incomplete block is carried
// into the next pass), together with each block's panel-relative byte offset. Per panel the work is
// O(entries + K / 32) shared-memory operations and no global atomics. k_emit_hub writes the blocks and values
// once the global scan has placed the panel.
constexpr int kHubThreads = 512;
#ifndef HRPB_EMIT_NT
#define HRPB_EMIT_NT 128
#endif
constexpr int kEmitNT = HRPB_EMIT_NT;  // threads of k_emit (listed panels; a CTA per panel, latency-bound: 128
                                       // threads at 16 CTAs per SM keep twice the panels in flight of 256 at 8:
                                       // c3 k_emit 0.46 -> 0.35 ms, c5 build 1.08 -> 1.02 ms)
constexpr int kEmitHubNT = 256;        // threads of k_emit_hub (the K > 2^23 hub path)
constexpr int kHubPassWords = 32768;                 // bitmap words per pass
constexpr int64_t kHubPassCols = 32 * kHubPassWords;  // 2^20 columns per pass
constexpr int kHubGroups = kHubPassWords / 8;        // 4096 groups of 8 words (u8 prefix within a group)
constexpr int kHubPatSlots = 2048;                   // brick-pattern window (u64 slots)
constexpr int kHubBndWords = 1024;                   // per-row pass boundaries: TM x (passes + 1) <= this
constexpr int kHubU = 4;                             // entries per thread in flight in the entry loops
constexpr int kHubMetaChunk = 256;                   // blocks per metadata work item of k_emit_hub
constexpr int kHubEntryChunk = 4096;                 // entries per value work item of k_emit_hub
struct HubSmem {
  uint32_t bits[kHubPassWords];
  uint8_t pre8[kHubPassWords];  // popcount of the earlier words of the word's 8-word group (<= 224)
  uint32_t gpre[kHubGroups];    // ranks before the group (panel-wide)
  unsigned long long pat[kHubPatSlots];
  uint32_t bnd[kHubBndWords];  // bnd[r * (npass + 1) + k] = first entry (panel-relative) of row r in pass >= k
  uint32_t off[129];           // pass entries: exclusive prefix over rows
  int64_t rp[129];
  uint32_t scan[kHubThreads / 32 + 1];
  uint32_t t;
};
__host__ __device__ inline bool hub_dense_ok(int64_t K, int tm) {
  return (int64_t)tm * (ceil_div(K, kHubPassCols) + 1) <= kHubBndWords;
}
__device__ __forceinline__ int64_t rel_base(int64_t e0, int64_t p, int tk) { return e0 / tk + 2 * p; }

// row of flattened pass item i: largest r with off[r] <= i (off[0] = 0, nondecreasing)
__device__ __forceinline__ int hub_row_of(const uint32_t* off, int nrows, uint32_t i) {
  int lo = 0, hi = nrows - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (off[mid] <= i) lo = mid; else hi = mid - 1;
  }
  return lo;
}

__global__ void __launch_bounds__(kHubThreads) k_count_hub(const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                          int64_t nnz, int tm, int tk, uint32_t* __restrict__ q,
                                                          uint32_t* __restrict__ nact_out,
                                                          uint32_t* __restrict__ nblk_out,
                                                          uint32_t* __restrict__ pbytes_out,
                                                          uint64_t* __restrict__ gpat, uint32_t* __restrict__ relb,
                                                          const uint32_t* __restrict__ biglist,
                                                          const uint32_t* __restrict__ nbig, uint32_t* work,
                                                          uint32_t* __restrict__ hublist, uint32_t* __restrict__ hubch,
                                                          unsigned long long* __restrict__ nhub, uint32_t* status) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t dsm[];
  HubSmem& S = *reinterpret_cast<HubSmem*>(dsm);
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t count = *nbig;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const int npass = (int)ceil_div(K, kHubPassCols);
  const int cap_blk = kHubPatSlots / nbk;  // blocks in the pattern window
  const int tk_sh = tk == 16 ? 4 : 5;
  while (true) {
    if (tid == 0) S.t = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t t = S.t;
    if (t >= count) break;
    const int64_t p = biglist[t];
    load_panel_rows(rp, M, nnz, tm, p, S.rp, status);  // (barriers)
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = S.rp[0], e1 = S.rp[nrows];
    const int nb1 = npass + 1;
    // (1) validation and the per-row pass boundaries: entry e starts pass k's range of its row for every
    // k in (pass(e - 1), pass(e)] (the row's first entry: k in [0, pass(e)]); rows end at their last pass
    for (int r = tid; r < nrows; r += kHubThreads) {
      const uint32_t b = (uint32_t)(S.rp[r] - e0), e = (uint32_t)(S.rp[r + 1] - e0);
      S.bnd[r * nb1 + npass] = e;
      if (b == e)
        for (int k = 0; k < npass; ++k) S.bnd[r * nb1 + k] = e;
    }
    __syncthreads();
    bool bad_range = false, bad_order = false;
    for (int64_t eb = e0; eb < e1; eb += kHubThreads * kHubU) {
     int32_t cvs[kHubU], cps[kHubU];
#pragma unroll
     for (int u = 0; u < kHubU; ++u) {  // (kHubU entries' loads in flight per thread)
       const int64_t e = eb + u * kHubThreads + tid;
       cvs[u] = e < e1 ? ci[e] : 0;
       cps[u] = e < e1 && e > e0 ? ci[e - 1] : 0;
     }
#pragma unroll
     for (int u = 0; u < kHubU; ++u) {
      const int64_t e = eb + u * kHubThreads + tid;
      if (e >= e1) continue;
      const int32_t c = cvs[u];
      if (c < 0 || c >= K) bad_range = true;
      const int r = row_of(S.rp, nrows, e);
      const bool first = e == S.rp[r];
      const int32_t cp = first ? 0 : cps[u];
      if (!first && cp >= c) bad_order = true;
      const int kc = (int)(min(max(c, 0), (int32_t)(K - 1)) / kHubPassCols);
      const int kp = first ? -1 : (int)(min(max(cp, 0), (int32_t)(K - 1)) / kHubPassCols);
      // (an unsorted row may step back: kc < kp then sets nothing; its entries are still clamped into range)
      for (int k = kp + 1; k <= kc; ++k) S.bnd[r * nb1 + k] = (uint32_t)(e - e0);
      if (e + 1 == S.rp[r + 1])  // last entry: the row has nothing in later passes
        for (int k = kc + 1; k < npass; ++k) S.bnd[r * nb1 + k] = (uint32_t)(e + 1 - e0);
     }
    }
    if (__any_sync(0xffffffffu, bad_range) && lane == 0) atomicOr(status, ST_COL_RANGE);
    if (__any_sync(0xffffffffu, bad_order) && lane == 0) atomicOr(status, ST_COL_ORDER);
    __syncthreads();
    uint32_t base = 0;         // ranks of earlier passes
    uint32_t jw = 0;           // first block of the pattern window (blocks < jw are flushed; jw may hold carried bits)
    uint32_t bytes = 0;        // panel-relative byte offset of block jw
    for (int i = tid; i < cap_blk * nbk; i += kHubThreads) S.pat[i] = 0ull;
    uint32_t* rel = relb + rel_base(e0, p, tk);
    unsigned long long* gp = reinterpret_cast<unsigned long long*>(gpat + pat_base(e0, p, nbk, tk));
    for (int k = 0; k < npass; ++k) {
      // entries of pass k: rows' ranges [bnd[r][k], bnd[r][k+1]), flattened by an exclusive prefix over rows
      if (tid < 32) {
        uint32_t carry = 0;
        for (int r0 = 0; r0 < nrows; r0 += 32) {
          const int r = r0 + lane;
          uint32_t len = 0;
          if (r < nrows) {
            const uint32_t b = S.bnd[r * nb1 + k], e = S.bnd[r * nb1 + k + 1];
            len = e > b ? e - b : 0u;
          }
          uint32_t tot;
          const uint32_t ex = warp_excl_scan(len, &tot);
          if (r < nrows) S.off[r] = carry + ex;
          carry += tot;
        }
        if (lane == 0) S.off[nrows] = carry;
      }
      __syncthreads();
      const uint32_t npe = S.off[nrows];
      const bool last = k == npass - 1;
      if (npe == 0 && !last) continue;  // (CTA-uniform)
      const int64_t c0 = (int64_t)k * kHubPassCols;
      for (int i = tid; i < kHubPassWords; i += kHubThreads) S.bits[i] = 0u;
      __syncthreads();
      for (uint32_t i0 = 0; i0 < npe; i0 += kHubThreads * kHubU) {  // set bits (kHubU loads in flight per thread)
        int32_t cv[kHubU];
#pragma unroll
        for (int u = 0; u < kHubU; ++u) {
          const uint32_t i = i0 + u * kHubThreads + tid;
          cv[u] = -1;
          if (i < npe) {
            const int r = hub_row_of(S.off, nrows, i);
            cv[u] = ci[e0 + S.bnd[r * nb1 + k] + (i - S.off[r])];
          }
        }
#pragma unroll
        for (int u = 0; u < kHubU; ++u) {
          if (i0 + u * kHubThreads + tid >= npe) continue;
          const int64_t c = min(max((int64_t)cv[u], (int64_t)0), K - 1) - c0;
          const uint32_t w = (uint32_t)min(max(c, (int64_t)0), kHubPassCols - 1);
          atomicOr(&S.bits[w >> 5], 1u << (w & 31));
        }
      }
      __syncthreads();
      {  // warp w: groups [256 w, 256 w + 256) of 8 words, 32 at a time (lane = group, two conflict-free 128-bit
         // loads): u8 prefix per word, group totals scanned across the warp, warp totals across the CTA
        constexpr int GPW = kHubGroups / (kHubThreads / 32);  // groups per warp (256)
        const int w = tid >> 5;
        uint32_t gsum[GPW / 32];
#pragma unroll
        for (int h = 0; h < GPW / 32; ++h) {
          const int g = w * GPW + h * 32 + lane;
          const uint4 a = *reinterpret_cast<const uint4*>(&S.bits[8 * g]);
          const uint4 b = *reinterpret_cast<const uint4*>(&S.bits[8 * g + 4]);
          const uint32_t c[8] = {(uint32_t)__popc(a.x), (uint32_t)__popc(a.y), (uint32_t)__popc(a.z),
                                 (uint32_t)__popc(a.w), (uint32_t)__popc(b.x), (uint32_t)__popc(b.y),
                                 (uint32_t)__popc(b.z), (uint32_t)__popc(b.w)};
          uint32_t run = 0, lo = 0, hi = 0;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (i < 4) lo |= run << (8 * i); else hi |= run << (8 * (i - 4));
            run += c[i];
          }
          *reinterpret_cast<uint2*>(&S.pre8[8 * g]) = make_uint2(lo, hi);
          gsum[h] = run;
        }
        uint32_t incl[GPW / 32];  // inclusive scans across the warp, the 8 rounds interleaved
#pragma unroll
        for (int h = 0; h < GPW / 32; ++h) incl[h] = gsum[h];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
          for (int h = 0; h < GPW / 32; ++h) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, incl[h], o);
            if (lane >= o) incl[h] += y;
          }
        }
        uint32_t wtot = 0, hbase[GPW / 32];
#pragma unroll
        for (int h = 0; h < GPW / 32; ++h) {
          hbase[h] = wtot;
          wtot += __shfl_sync(0xffffffffu, incl[h], 31);
        }
        uint32_t tot;
        const uint32_t wex = block_excl_scan<kHubThreads>(lane == 0 ? wtot : 0u, &tot, S.scan);
        const uint32_t wbase = base + __shfl_sync(0xffffffffu, wex, 0);
#pragma unroll
        for (int h = 0; h < GPW / 32; ++h) S.gpre[w * GPW + h * 32 + lane] = wbase + hbase[h] + incl[h] - gsum[h];
        __syncthreads();
        // ranks (in the panel) of the pass's entries, and their brick-pattern bits: blocks in the shared window
        // [jw, jw + cap_blk) by shared atomics, later blocks (huge passes) by global atomics into gp
        const uint32_t jend = (base + tot + tk - 1) >> tk_sh;  // blocks touched after this pass
        const uint32_t jwe = jw + cap_blk;
        for (uint32_t j = max(jw, jwe) + tid; j < jend; j += kHubThreads)  // (beyond the window: zero, then OR)
          for (int i = 0; i < nbk; ++i) gp[(int64_t)j * nbk + i] = 0ull;
        __syncthreads();
        for (uint32_t i0 = 0; i0 < npe; i0 += kHubThreads * kHubU) {
         int rr[kHubU];
         uint32_t ee[kHubU];
         int32_t cv[kHubU];
#pragma unroll
         for (int u = 0; u < kHubU; ++u) {  // (kHubU entries' loads in flight per thread)
           const uint32_t i = i0 + u * kHubThreads + tid;
           rr[u] = 0;
           ee[u] = 0;
           cv[u] = 0;
           if (i < npe) {
             rr[u] = hub_row_of(S.off, nrows, i);
             ee[u] = S.bnd[rr[u] * nb1 + k] + (i - S.off[rr[u]]);
             cv[u] = ci[e0 + ee[u]];
           }
         }
#pragma unroll
         for (int u = 0; u < kHubU; ++u) {
          if (i0 + u * kHubThreads + tid >= npe) continue;
          const int r = rr[u];
          const uint32_t e = ee[u];
          const int64_t c = min(max((int64_t)cv[u], (int64_t)0), K - 1) - c0;
          const uint32_t w = (uint32_t)min(max(c, (int64_t)0), kHubPassCols - 1), wd = w >> 5;
          const uint32_t qq = S.gpre[wd >> 3] + S.pre8[wd] + __popc(S.bits[wd] & ((1u << (w & 31)) - 1u));
          q[e0 + e] = qq;
          const uint32_t j = qq >> tk_sh, lc = qq & (tk - 1);
          const int bit = ((r & 15) << 2) | (int)(lc & 3);
          const int slot = (int)(lc >> 2) * nbrow + (r >> 4);
          if (j < jwe) {
            uint32_t* half = reinterpret_cast<uint32_t*>(&S.pat[(j - jw) * nbk + slot]) + (bit >> 5);
            atomicOr(half, 1u << (bit & 31));
          } else {
            atomicOr(&gp[(int64_t)j * nbk + slot], 1ull << bit);
          }
         }
        }
        base += tot;
      }
      __threadfence_block();
      __syncthreads();
      // flush the blocks complete after this pass: patterns (window blocks from shared memory), sizes, relative
      // offsets; the pass's incomplete last block is carried into the window's slot 0
      const uint32_t jend = (base + tk - 1) >> tk_sh;
      const uint32_t jcomplete = last ? jend : (base >> tk_sh);
      const uint32_t jwe = jw + cap_blk;
      for (uint32_t c2 = jw; c2 < jcomplete; c2 += kHubThreads) {
        const uint32_t j = c2 + tid;
        uint32_t size = 0;
        if (j < jcomplete) {
          uint32_t nbr = 0, nz = 0;
          for (int i = 0; i < nbk; ++i) {
            unsigned long long v;
            if (j < jwe) {
              v = S.pat[(j - jw) * nbk + i];
              gp[(int64_t)j * nbk + i] = v;
            } else {
              v = __ldcg(&gp[(int64_t)j * nbk + i]);
            }
            nbr += v != 0ull;
            nz += __popcll(v);
          }
          size = block_bytes(nbc, nbr, nz);
        }
        uint32_t tot;
        const uint32_t ex = block_excl_scan<kHubThreads>(size, &tot, S.scan);
        if (j < jcomplete) rel[j] = bytes + ex;
        bytes += tot;
      }
      __syncthreads();
      if (jcomplete < jend) {  // carry block jcomplete
        unsigned long long keep = 0ull;
        if (tid < nbk)
          keep = jcomplete < jwe ? S.pat[(jcomplete - jw) * nbk + tid] : __ldcg(&gp[(int64_t)jcomplete * nbk + tid]);
        __syncthreads();
        for (int i = tid; i < cap_blk * nbk; i += kHubThreads) S.pat[i] = i < nbk ? keep : 0ull;
      } else {
        for (int i = tid; i < cap_blk * nbk; i += kHubThreads) S.pat[i] = 0ull;
      }
      jw = jcomplete;
      __syncthreads();
    }
    const uint32_t nact = base, nblk = (nact + tk - 1) >> tk_sh;
    if (tid == 0) {
      nact_out[p] = nact;
      nblk_out[p] = nblk;
      pbytes_out[p] = bytes;
      // work items of k_emit_hub: block-metadata chunks, then value chunks
      const unsigned long long items =
          (unsigned long long)(ceil_div(nblk, kHubMetaChunk) + ceil_div(e1 - e0, kHubEntryChunk));
      const unsigned long long old = atomicAdd(nhub, (1ull << 32) + items);
      hublist[old >> 32] = (uint32_t)p;
      hubch[old >> 32] = (uint32_t)old;
    }
  }
}

// ------------------------------------------------------------------ hub panels, two-level bitmap (K <= 2^23)
// One CTA per hub panel (claimed dynamically). Ranks (R23: ascending distinct columns) from a two-level
// bitmap over the whole column space instead of dense passes: occ2 holds one bit per 32-column word, the occupied
// words get dense ordinals (popcount prefix over occ2), mask[ordinal] collects the word's column bits and
// mpre[ordinal] = ranks before the word, so rank = mpre[o] + popc(mask[o] & lower bits). Work per panel is
// O(entries + K / 1024) shared-memory operations: three passes over the entries (word bits; column bits; ranks and
// brick patterns) plus two prefix scans. Entries are staged in shared memory when they fit (kH2Stage), the masks
// when the occupied words fit (kH2OrdCap, else this CTA's global scratch). Brick patterns of the first blocks
// go to a shared-memory window, later blocks to global memory by atomics. Outputs as k_count_hub (q, patterns,
// block-relative byte offsets, counts, k_emit_hub work items).
#ifndef HRPB_H2_THREADS
#define HRPB_H2_THREADS 1024  // (512: c3 hub 1.84 ms, 1024: 1.57 ms)
#endif
constexpr int kH2Threads = HRPB_H2_THREADS;
#ifndef HRPB_H2_MINB
#define HRPB_H2_MINB 1             // CTAs per SM (2 with 4096-entry caps: c3 hub 2.03 -> 2.34 ms)
#endif
constexpr int kH2OccWords = 8192;  // one bit per 32-column word: K <= 2^23
constexpr int kH2OrdCap = 8192;    // occupied words whose masks stay in shared memory
#ifndef HRPB_H2_STAGE
#define HRPB_H2_STAGE 8192
#endif
constexpr int kH2Stage = HRPB_H2_STAGE;  // entries staged in shared memory
constexpr int kH2PatSlots = 2048;  // brick-pattern window (u64 slots)
constexpr int64_t kH2Huge = 65536; // panels with more entries are claimed first (the critical path of the kernel)
#ifndef HRPB_E2_THREADS
#define HRPB_E2_THREADS 512
#endif
constexpr int kE2Threads = HRPB_E2_THREADS;  // k_emit_hub2 threads (one per block of a work item at nbk = 4)
constexpr int kE2Slots = 4 * kE2Threads;     // brick slots (blocks x TM/16 x TK/4) per k_emit_hub2 work item
constexpr int kE2MinB = 1536 / kE2Threads;   // k_emit_hub2 CTAs per SM
#ifndef HRPB_H2_U
#define HRPB_H2_U 4
#endif
constexpr int kH2U = HRPB_H2_U;    // entries per thread in flight in the global entry loops
struct Hub2Smem {
  uint32_t occ2[kH2OccWords];
  uint32_t opre[kH2OccWords];
  uint32_t mask[kH2OrdCap];
  uint32_t mpre[kH2OrdCap];
  uint32_t col[kH2Stage];
  unsigned long long pat[kH2PatSlots];
  uint8_t row[kH2Stage];
  int64_t rp[129];
  uint32_t scan[kH2Threads / 32 + 1];
  uint32_t t;
};
__host__ __device__ inline bool hub2_ok(int64_t K) { return K <= 32ll * 32 * kH2OccWords; }

__global__ void __launch_bounds__(kH2Threads, HRPB_H2_MINB) k_count_hub2(const int64_t* __restrict__ rp,
                                                             const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                             int64_t nnz, int tm, int tk, uint32_t* __restrict__ q,
                                                             uint32_t* __restrict__ nact_out,
                                                             uint32_t* __restrict__ nblk_out,
                                                             uint32_t* __restrict__ pbytes_out,
                                                             uint64_t* __restrict__ gpat, uint32_t* __restrict__ relb,
                                                             const uint32_t* __restrict__ biglist,
                                                             const uint32_t* __restrict__ nbig, uint32_t* work,
                                                             uint32_t* __restrict__ hublist,
                                                             uint32_t* __restrict__ hubch,
                                                             unsigned long long* __restrict__ nhub,
                                                             uint32_t* __restrict__ scratch, uint32_t* status,
                                                             const uint32_t* __restrict__ nhuge, int64_t P) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t dsm[];
  Hub2Smem& S = *reinterpret_cast<Hub2Smem*>(dsm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t nh = *nhuge, count = *nbig + nh;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const int tk_sh = tk == 16 ? 4 : 5;
  const int cap_blk = kH2PatSlots / nbk;  // blocks in the pattern window
  const int64_t W = ceil_div(K, 32);      // 32-column words
  uint32_t* const gmask = scratch + (size_t)blockIdx.x * 2 * W;  // masks / prefixes beyond kH2OrdCap words
  uint32_t* const gmpre = gmask + W;
  constexpr int kPer = kH2OccWords / kH2Threads;  // occupancy words per thread in the prefix scan (16)
  for (int i = tid; i < kH2OccWords / 4; i += kH2Threads) reinterpret_cast<uint4*>(S.occ2)[i] = make_uint4(0, 0, 0, 0);
  while (true) {
    if (tid == 0) S.t = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t t = S.t;
    if (t >= count) break;
    const int64_t p = t < nh ? biglist[P - t] : biglist[t - nh];  // the largest panels first (listed from the end)
    load_panel_rows(rp, M, nnz, tm, p, S.rp, status);  // (barriers: also orders S.t's read and occ2's clearing)
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = S.rp[0], e1 = S.rp[nrows];
    const uint32_t E = (uint32_t)(e1 - e0);
    const bool staged = E <= (uint32_t)kH2Stage;
    // (1) validation, staging, word-occupancy bits; each thread's entries ascend, so its row only
    // moves forward
    {
      bool bad_range = false, bad_order = false;
      int r = 0;
      for (uint32_t i0 = 0; i0 < E; i0 += kH2Threads * kH2U) {
        int32_t cv[kH2U], pv[kH2U];
#pragma unroll
        for (int u = 0; u < kH2U; ++u) {
          const uint32_t i = i0 + u * kH2Threads + tid;
          cv[u] = i < E ? ci[e0 + i] : 0;
          pv[u] = (lane == 0 && i < E && i > 0) ? ci[e0 + i - 1] : 0;
        }
#pragma unroll
        for (int u = 0; u < kH2U; ++u) {
          const uint32_t i = i0 + u * kH2Threads + tid;
          const int32_t up = __shfl_up_sync(0xffffffffu, cv[u], 1);  // entry i - 1 (lane 0: loaded)
          if (i >= E) continue;
          const int64_t e = e0 + i;
          while (S.rp[r + 1] <= e) ++r;
          const int32_t c = cv[u];
          if (c < 0 || c >= K) bad_range = true;
          if (e != S.rp[r] && (lane ? up : pv[u]) >= c) bad_order = true;
          const uint32_t cc = (uint32_t)min(max(c, 0), (int32_t)(K - 1));
          if (staged) {
            S.col[i] = cc;
            S.row[i] = (uint8_t)r;
          }
          const uint32_t w = cc >> 5;
          atomicOr(&S.occ2[w >> 5], 1u << (w & 31));
        }
      }
      if (__any_sync(0xffffffffu, bad_range) && lane == 0) atomicOr(status, ST_COL_RANGE);
      if (__any_sync(0xffffffffu, bad_order) && lane == 0) atomicOr(status, ST_COL_ORDER);
    }
    __syncthreads();
    // (2) dense ordinals of the occupied words (thread: kPer consecutive occupancy words)
    uint32_t nocc;
    {
      uint32_t cnt[kPer], sum = 0;
#pragma unroll
      for (int k = 0; k < kPer / 4; ++k) {
        const uint4 v = reinterpret_cast<const uint4*>(S.occ2)[tid * (kPer / 4) + k];
        cnt[4 * k] = __popc(v.x); cnt[4 * k + 1] = __popc(v.y); cnt[4 * k + 2] = __popc(v.z); cnt[4 * k + 3] = __popc(v.w);
      }
#pragma unroll
      for (int k = 0; k < kPer; ++k) sum += cnt[k];
      uint32_t run = block_excl_scan<kH2Threads>(sum, &nocc, S.scan);
#pragma unroll
      for (int k = 0; k < kPer / 4; ++k) {
        uint4 v;
        v.x = run; run += cnt[4 * k];
        v.y = run; run += cnt[4 * k + 1];
        v.z = run; run += cnt[4 * k + 2];
        v.w = run; run += cnt[4 * k + 3];
        reinterpret_cast<uint4*>(S.opre)[tid * (kPer / 4) + k] = v;
      }
    }
    const bool in_smem = nocc <= (uint32_t)kH2OrdCap;
    uint32_t* const mask = in_smem ? S.mask : gmask;
    uint32_t* const mpre = in_smem ? S.mpre : gmpre;
    for (uint32_t o = tid; o < nocc; o += kH2Threads) mask[o] = 0u;
    __syncthreads();
    auto ordinal = [&](uint32_t c) {
      const uint32_t w = c >> 5;
      return S.opre[w >> 5] + __popc(S.occ2[w >> 5] & ((1u << (w & 31)) - 1u));
    };
    // (3) column bits of the occupied words
    if (staged) {
      for (uint32_t i = tid; i < E; i += kH2Threads) {
        const uint32_t c = S.col[i];
        atomicOr(&mask[ordinal(c)], 1u << (c & 31));  // (shared memory unless nocc > kH2OrdCap)
      }
    } else {
      for (uint32_t i0 = 0; i0 < E; i0 += kH2Threads * kH2U) {
        int32_t cv[kH2U];
#pragma unroll
        for (int u = 0; u < kH2U; ++u) {
          const uint32_t i = i0 + u * kH2Threads + tid;
          cv[u] = i < E ? ci[e0 + i] : 0;
        }
#pragma unroll
        for (int u = 0; u < kH2U; ++u) {
          if (i0 + u * kH2Threads + tid >= E) continue;
          const uint32_t c = (uint32_t)min(max(cv[u], 0), (int32_t)(K - 1));
          atomicOr(&mask[ordinal(c)], 1u << (c & 31));
        }
      }
    }
    __syncthreads();
    // (4) ranks before each occupied word: warp w scans a contiguous range of ordinals, 32 consecutive at a time
    uint32_t nact;
    {
      constexpr int kWarps = kH2Threads / 32;
      const uint32_t per = ((nocc + kWarps - 1) / kWarps + 31) & ~31u;
      const uint32_t o0 = min((uint32_t)warp * per, nocc), o1 = min(o0 + per, nocc);
      uint32_t sum = 0;
#pragma unroll 4
      for (uint32_t o = o0 + lane; o < o1; o += 32) sum += __popc(mask[o]);
#pragma unroll
      for (int k = 16; k; k >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, k);
      uint32_t run = block_excl_scan<kH2Threads>(lane == 0 ? sum : 0u, &nact, S.scan);
      run = __shfl_sync(0xffffffffu, run, 0);
      for (uint32_t ob = o0; ob < o1; ob += 32) {
        const uint32_t o = ob + lane;
        const uint32_t v = o < o1 ? __popc(mask[o]) : 0u;
        uint32_t x = v;
#pragma unroll
        for (int k = 1; k < 32; k <<= 1) {
          const uint32_t y = __shfl_up_sync(0xffffffffu, x, k);
          if (lane >= k) x += y;
        }
        if (o < o1) mpre[o] = run + x - v;
        run += __shfl_sync(0xffffffffu, x, 31);
      }
    }
    const uint32_t nblk = (nact + tk - 1) >> tk_sh;
    unsigned long long* gp = reinterpret_cast<unsigned long long*>(gpat + pat_base(e0, p, nbk, tk));
    for (int i = tid; i < cap_blk * nbk; i += kH2Threads) S.pat[i] = 0ull;
    for (int64_t i = (int64_t)cap_blk * nbk + tid; i < (int64_t)nblk * nbk; i += kH2Threads) gp[i] = 0ull;
    __syncthreads();
    // (5) ranks and brick patterns (bit (r % 16) * 4 + q % 4 of brick (q % TK / 4, r / 16), R3 / R4)
    auto rank_entry = [&](uint32_t i, uint32_t c, int r) {
      const uint32_t o = ordinal(c);
      const uint32_t qq = mpre[o] + __popc(mask[o] & ((1u << (c & 31)) - 1u));
      q[e0 + i] = qq;
      const uint32_t j = qq >> tk_sh, lc = qq & (tk - 1);
      const int bit = ((r & 15) << 2) | (int)(lc & 3);
      const int slot = (int)(lc >> 2) * nbrow + (r >> 4);
      if (j < (uint32_t)cap_blk)
        atomicOr(reinterpret_cast<uint32_t*>(&S.pat[j * nbk + slot]) + (bit >> 5), 1u << (bit & 31));
      else
        atomicOr(&gp[(int64_t)j * nbk + slot], 1ull << bit);
    };
    if (staged) {
      for (uint32_t i = tid; i < E; i += kH2Threads) rank_entry(i, S.col[i], S.row[i]);
    } else {
      int r = 0;
      for (uint32_t i0 = 0; i0 < E; i0 += kH2Threads * kH2U) {
        int32_t cv[kH2U];
#pragma unroll
        for (int u = 0; u < kH2U; ++u) {
          const uint32_t i = i0 + u * kH2Threads + tid;
          cv[u] = i < E ? ci[e0 + i] : 0;
        }
#pragma unroll
        for (int u = 0; u < kH2U; ++u) {
          const uint32_t i = i0 + u * kH2Threads + tid;
          if (i >= E) continue;
          while (S.rp[r + 1] <= e0 + (int64_t)i) ++r;
          rank_entry(i, (uint32_t)min(max(cv[u], 0), (int32_t)(K - 1)), r);
        }
      }
    }
    __threadfence();
    __syncthreads();
    // (6) block sizes and panel-relative byte offsets; the window's patterns go out to global memory
    uint32_t* rel = relb + rel_base(e0, p, tk);
    uint32_t bytes = 0;
    for (uint32_t c2 = 0; c2 < nblk; c2 += kH2Threads) {
      const uint32_t j = c2 + tid;
      uint32_t size = 0;
      if (j < nblk) {
        uint32_t nbr = 0, nz = 0;
        for (int i = 0; i < nbk; ++i) {
          unsigned long long v;
          if (j < (uint32_t)cap_blk) {
            v = S.pat[j * nbk + i];
            gp[(int64_t)j * nbk + i] = v;
          } else {
            v = __ldcg(&gp[(int64_t)j * nbk + i]);
          }
          nbr += v != 0ull;
          nz += __popcll(v);
        }
        size = block_bytes(nbc, nbr, nz);
      }
      uint32_t tot;
      const uint32_t ex = block_excl_scan<kH2Threads>(size, &tot, S.scan);
      if (j < nblk) rel[j] = bytes + ex;
      bytes += tot;
    }
    __syncthreads();
    for (int i = tid; i < kH2OccWords / 4; i += kH2Threads) reinterpret_cast<uint4*>(S.occ2)[i] = make_uint4(0, 0, 0, 0);
    if (tid == 0) {
      nact_out[p] = nact;
      nblk_out[p] = nblk;
      pbytes_out[p] = bytes;
      const unsigned long long items = (unsigned long long)ceil_div(nblk, kE2Slots / nbk);  // k_emit_hub2 items
      const unsigned long long old = atomicAdd(nhub, (1ull << 32) + items);
      hublist[old >> 32] = (uint32_t)p;
      hubch[old >> 32] = (uint32_t)old;
    }
  }
}

// Hub panels' output (after k_count_hub2 and the global scan), in block order: work item = kE2Slots / nbk
// consecutive blocks of one hub. The item stages its blocks' patterns in shared memory, writes their sizePtr,
// HRPB-v1 headers, patterns and padding, then finds in every row the entries whose ranks fall in its blocks (one
// contiguous range per row: ranks ascend along a row, R23) and writes their activeCols and values at popcount
// ranks — the stores of an item land in one contiguous output region.
constexpr int kE2U = 4;  // entries per thread in flight
__global__ void __launch_bounds__(kE2Threads, kE2MinB) k_emit_hub2(const int64_t* __restrict__ rp,
                                                         const int32_t* __restrict__ ci,
                                                         const float* __restrict__ vals, int64_t M, int64_t K,
                                                         int64_t nnz, int tm, int tk, const uint32_t* __restrict__ q,
                                                         const uint32_t* __restrict__ nact_in,
                                                         const uint32_t* __restrict__ brp,
                                                         const uint64_t* __restrict__ poff,
                                                         const uint64_t* __restrict__ gpat,
                                                         const uint32_t* __restrict__ relb, uint32_t* __restrict__ ac,
                                                         uint64_t* __restrict__ sp, uint8_t* __restrict__ packed,
                                                         const uint32_t* __restrict__ hublist,
                                                         const uint32_t* __restrict__ hubch,
                                                         const unsigned long long* __restrict__ nhub) {
  pdl_wait();
  __shared__ int64_t s_rp[129];
  __shared__ unsigned long long s_pt[kE2Slots];
  __shared__ uint16_t s_so[kE2Slots];
  __shared__ uint64_t s_vb[kE2Slots / 4];
  __shared__ uint32_t s_seg[128];
  __shared__ uint32_t s_off[129];
  __shared__ uint32_t s_hub;
  const unsigned long long hc = *nhub;
  const uint32_t count = (uint32_t)(hc >> 32), total = (uint32_t)hc;
  const int tid = threadIdx.x;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const int tk_sh = tk == 16 ? 4 : 5;
  const uint32_t bpi = (uint32_t)(kE2Slots / nbk);  // blocks per item
  for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
    if (tid < 32) {  // last hub t with hubch[t] <= g: 32-way search by warp 0
      uint32_t lo = 0, n = count;
      while (n > 1) {
        const uint32_t step = (n + 31) / 32;
        const uint32_t i = lo + tid * step;
        const bool le = i < lo + n && hubch[i] <= g;
        const uint32_t k = 31 - __clz(__ballot_sync(0xffffffffu, le) | 1u);
        lo += k * step;
        n = min(step, n - k * step);
      }
      if (tid == 0) s_hub = lo;
    }
    __syncthreads();
    const uint32_t hub = s_hub;
    const int64_t p = hublist[hub];
    const uint32_t item = g - hubch[hub];
    load_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);  // (barriers)
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = s_rp[0];
    const uint32_t b0 = brp[p], nblk = brp[p + 1] - b0, nact = nact_in[p];
    const uint64_t pbase = poff[p];
    const uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
    const uint32_t* rel = relb + rel_base(e0, p, tk);
    const uint32_t j0 = item * bpi, j1 = min(j0 + bpi, nblk), nb = j1 > j0 ? j1 - j0 : 0u;
    for (uint32_t i = tid; i < nb * nbk; i += kE2Threads) s_pt[i] = gp[(int64_t)j0 * nbk + i];
    {  // row r (warp r % 16): its entries with ranks in [j0 TK, j1 TK), by 32-way lower-bound searches on the
       // ascending ranks of the row (~3 dependent loads per search)
      const int lane = tid & 31;
      for (int r = tid >> 5; r < nrows; r += kE2Threads / 32) {
        const int64_t rb = s_rp[r], re = s_rp[r + 1];
        auto lower = [&](uint32_t x) {  // first e in [rb, re) with q[e] >= x
          int64_t lo = rb, n = re - rb;  // answer in [lo, lo + n]
          while (n > 0) {
            const int64_t step = (n + 31) / 32;
            const int64_t i = lo + (int64_t)lane * step;
            const bool lt = i < lo + n && q[i] < x;
            const int k = __popc(__ballot_sync(0xffffffffu, lt));  // probes below x (a prefix of the lanes)
            if (k == 0) break;
            lo += (int64_t)(k - 1) * step + 1;
            n = min(step - 1, re - lo);
          }
          return lo;
        };
        const int64_t a = lower(j0 << tk_sh), b = max(a, lower(j1 << tk_sh));
        if (lane == 0) {
          s_seg[r] = (uint32_t)(a - e0);
          s_off[r] = (uint32_t)(b - a);
        }
      }
    }
    __syncthreads();
    if (tid < 32) {  // flattened entry ranges: exclusive prefix over the rows
      uint32_t carry = 0;
      for (int r0 = 0; r0 < nrows; r0 += 32) {
        const int r = r0 + tid;
        const uint32_t len = r < nrows ? s_off[r] : 0u;
        uint32_t tot;
        const uint32_t ex = warp_excl_scan(len, &tot);
        if (r < nrows) s_off[r] = carry + ex;
        carry += tot;
      }
      if (tid == 0) s_off[nrows] = carry;
    }
    if (tid < nb) {  // block j0 + tid: sizePtr, header, patterns, padding, its values' base and brick offsets
      const unsigned long long* pj = s_pt + tid * nbk;
      uint32_t nbr = 0, nz = 0;
      for (int i = 0; i < nbk; ++i) {
        s_so[tid * nbk + i] = (uint16_t)nz;
        nbr += pj[i] != 0ull;
        nz += __popcll(pj[i]);
      }
      const uint32_t j = j0 + tid;
      const uint64_t off = pbase + rel[j];
      sp[b0 + j] = off;
      emit_block_meta_dyn(packed + off, pj, nbc, nbrow, nbr, nz, block_bytes(nbc, nbr, nz));
      s_vb[tid] = off + ((nbc + 1 + nbr + 7) & ~7u) + 8 * nbr;
      if (j + 1 == nblk)
        for (uint32_t t = nact; t < nblk * (uint32_t)tk; ++t) ac[(int64_t)b0 * tk + t] = (uint32_t)K;
    }
    __syncthreads();
    const uint32_t ne = s_off[nrows];
    int r = 0;
    for (uint32_t i0 = 0; i0 < ne; i0 += kE2Threads * kE2U) {
      uint32_t qq[kE2U];
      int32_t cv[kE2U];
      float vv[kE2U];
      int rr[kE2U];
#pragma unroll
      for (int u = 0; u < kE2U; ++u) {
        const uint32_t i = i0 + u * kE2Threads + tid;
        qq[u] = 0xFFFFFFFFu;
        rr[u] = 0;
        if (i < ne) {
          while (s_off[r + 1] <= i) ++r;
          rr[u] = r;
          const int64_t e = e0 + s_seg[r] + (i - s_off[r]);
          qq[u] = q[e];
          cv[u] = ci[e];
          vv[u] = vals[e];
        }
      }
#pragma unroll
      for (int u = 0; u < kE2U; ++u) {
        const uint32_t jj = qq[u] >> tk_sh;
        if (qq[u] >= nact || jj < j0 || jj >= j1) continue;  // (only for invalid CSR input)
        const uint32_t jl = jj - j0, lc = qq[u] & (tk - 1);
        ac[((int64_t)b0 + jj) * tk + lc] = (uint32_t)cv[u];
        const int bit = ((rr[u] & 15) << 2) | (int)(lc & 3);
        const uint32_t slot = jl * nbk + (lc >> 2) * nbrow + (rr[u] >> 4);
        const uint32_t off = s_so[slot] + __popcll(s_pt[slot] & ((1ull << bit) - 1ull));
        reinterpret_cast<float*>(packed + s_vb[jl])[off] = vv[u];
      }
    }
  }
}

// Hub panels' output, after the global scan: every CTA takes items of one flat list (per hub: its block-metadata
// chunks — sizePtr = panel offset + relative offset, HRPB-v1 headers, patterns, padding, sentinel activeCols —
// then its 4096-entry value chunks — activeCols and values at popcount ranks).
__global__ void __launch_bounds__(kEmitHubNT) k_emit_hub(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                     const float* __restrict__ vals, int64_t M, int64_t K,
                                                     int64_t nnz, int tm, int tk, const uint32_t* __restrict__ q,
                                                     const uint32_t* __restrict__ nact_in,
                                                     const uint32_t* __restrict__ brp,
                                                     const uint64_t* __restrict__ poff,
                                                     const uint64_t* __restrict__ gpat,
                                                     const uint32_t* __restrict__ relb, uint32_t* __restrict__ ac,
                                                     uint64_t* __restrict__ sp, uint8_t* __restrict__ packed,
                                                     const uint32_t* __restrict__ hublist,
                                                     const uint32_t* __restrict__ hubch,
                                                     const unsigned long long* __restrict__ nhub) {
  pdl_wait();
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_hub;
  const unsigned long long hc = *nhub;
  const uint32_t count = (uint32_t)(hc >> 32), total = (uint32_t)hc;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const int tk_sh = tk == 16 ? 4 : 5;
  for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {
    if (threadIdx.x < 32) {  // last hub t with hubch[t] <= g: 32-way search by warp 0 (3 dependent loads at 12K hubs)
      const int lane = threadIdx.x;
      uint32_t lo = 0, n = count;  // answer in [lo, lo + n)
      while (n > 1) {
        const uint32_t step = (n + 31) / 32;
        const uint32_t i = lo + lane * step;
        const bool le = i < lo + n && hubch[i] <= g;
        const uint32_t k = 31 - __clz(__ballot_sync(0xffffffffu, le) | 1u);  // last probe <= g (probe 0 always is)
        lo += k * step;
        n = min(step, n - k * step);
      }
      if (lane == 0) s_hub = lo;
    }
    __syncthreads();
    const uint32_t hub = s_hub;
    const int64_t p = hublist[hub];
    const uint32_t item = g - hubch[hub];
    load_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);  // (barriers: also orders s_hub's reads before its reuse)
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = s_rp[0], e1 = s_rp[nrows];
    const uint32_t b0 = brp[p], nblk = brp[p + 1] - b0, nact = nact_in[p];
    const uint64_t pbase = poff[p];
    const uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
    const uint32_t* rel = relb + rel_base(e0, p, tk);
    const uint32_t nmeta = (uint32_t)ceil_div(nblk, kHubMetaChunk);
    if (item < nmeta) {
      const uint32_t j = item * kHubMetaChunk + threadIdx.x;
      if (j < nblk) {
        const unsigned long long* pj = reinterpret_cast<const unsigned long long*>(gp) + (int64_t)j * nbk;
        uint32_t nbr = 0, nz = 0;
        for (int i = 0; i < nbk; ++i) { nbr += pj[i] != 0ull; nz += __popcll(pj[i]); }
        const uint64_t off = pbase + rel[j];
        sp[b0 + j] = off;
        emit_block_meta_dyn(packed + off, pj, nbc, nbrow, nbr, nz, block_bytes(nbc, nbr, nz));
        if (j + 1 == nblk)
          for (uint32_t t = nact; t < nblk * (uint32_t)tk; ++t) ac[(int64_t)b0 * tk + t] = (uint32_t)K;
      }
      continue;
    }
    const int64_t c0e = e0 + (int64_t)(item - nmeta) * kHubEntryChunk;
    const int64_t c1e = min(e1, c0e + kHubEntryChunk);
    if (nbk == 4) {  // TM = TK = 16: kHubU entries per thread, each stage's loads issued before they are used
      int r = row_of(s_rp, nrows, c0e + threadIdx.x < c1e ? c0e + threadIdx.x : c0e);  // then only moves forward
      for (int64_t eb = c0e; eb < c1e; eb += kEmitHubNT * kHubU) {
        uint32_t qq[kHubU];
        int32_t cv[kHubU];
        float vv[kHubU];
#pragma unroll
        for (int u = 0; u < kHubU; ++u) {
          const int64_t e = eb + u * kEmitHubNT + threadIdx.x;
          qq[u] = 0xFFFFFFFFu;
          if (e < c1e) {
            qq[u] = q[e];
            cv[u] = ci[e];
            vv[u] = vals[e];
          }
        }
        uint64_t w[kHubU][4];
        uint32_t rl[kHubU];
#pragma unroll
        for (int u = 0; u < kHubU; ++u) {
          const uint32_t j = qq[u] < nact ? qq[u] >> tk_sh : 0u;
          const uint64_t* pt = gp + (int64_t)j * 4;
#pragma unroll
          for (int i = 0; i < 4; ++i) w[u][i] = pt[i];
          rl[u] = rel[j];
        }
#pragma unroll
        for (int u = 0; u < kHubU; ++u) {
          if (qq[u] >= nact) continue;  // (padding items; invalid CSR input)
          const int64_t e = eb + u * kEmitHubNT + threadIdx.x;
          while (s_rp[r + 1] <= e) ++r;
          const uint32_t j = qq[u] >> tk_sh, lc = qq[u] & (tk - 1);
          ac[((int64_t)b0 + j) * tk + lc] = (uint32_t)cv[u];
          const int bit = ((r & 15) << 2) | (lc & 3);
          const int mine = (int)(lc >> 2);
          uint32_t nbr = 0, off = 0;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            nbr += w[u][i] != 0ull;
            if (i < mine) off += __popcll(w[u][i]);
          }
          const uint64_t wm = mine == 0 ? w[u][0] : mine == 1 ? w[u][1] : mine == 2 ? w[u][2] : w[u][3];  // (no local)
          off += __popcll(wm & ((1ull << bit) - 1ull));
          const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
          reinterpret_cast<float*>(packed + pbase + rl[u] + hdr + 8 * nbr)[off] = vv[u];
        }
      }
      continue;
    }
    for (int64_t e = c0e + threadIdx.x; e < c1e; e += kEmitHubNT) {
      const uint32_t qq = q[e];
      const int32_t c = ci[e];
      const float v = vals[e];
      if (qq >= nact) continue;  // only for invalid CSR input
      const int r = row_of(s_rp, nrows, e);
      const uint32_t j = qq >> tk_sh, lc = qq & (tk - 1);
      ac[((int64_t)b0 + j) * tk + lc] = (uint32_t)c;
      const int bit = ((r & 15) << 2) | (lc & 3);
      const int mine = (lc >> 2) * nbrow + (r >> 4);
      const uint64_t* pt = gp + (int64_t)j * nbk;
      uint32_t nbr = 0, off = 0;
      for (int i = 0; i < nbk; ++i) {
        const uint64_t w = pt[i];
        nbr += w != 0ull;
        if (i < mine) off += __popcll(w);
      }
      off += __popcll(pt[mine] & ((1ull << bit) - 1ull));
      const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
      reinterpret_cast<float*>(packed + pbase + rel[j] + hdr + 8 * nbr)[off] = v;
    }
  }
}

// ------------------------------------------------------------------ pass B (CTA), listed panels
// One CTA per listed panel (claimed dynamically: listed panels differ in size by orders of magnitude). Block j of
// panel p is global block b0 + j (b0 = blockedRowPtr[p]); its byte offset is the panel offset plus the in-panel
// exclusive scan of block sizes (sizePtr). Header, patterns and values follow the HRPB-v1 layout; value
// destination = values base + popcount of the earlier bricks + popcount of the lower bits of its own brick
// (P:L211-219). Panels with <= kSmallCap entries stage their blocks' patterns, brick value offsets and value bases
// in shared memory and map entries to rows through a row map, so each entry costs its three coalesced loads (rank,
// column, value) and two stores; hub panels (> kHubEmit entries) only get their block metadata here, their values
// are scattered by every CTA in k_emit_hubvals.
__host__ __device__ constexpr size_t emit_smem_bytes(int tm, int tk) {
  return (size_t)(kSmallCap / tk + 1) * ((tk / HRPB_BRICK_K) * (tm / HRPB_BRICK_M) * 10 + 8) + kSmallCap + 64;
}

__global__ void __launch_bounds__(kEmitNT) k_emit(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                 const float* __restrict__ vals, int64_t M, int64_t K,
                                                 int64_t nnz, int tm, int tk, const uint32_t* __restrict__ q,
                                                 const uint32_t* __restrict__ nact_in,
                                                 const uint32_t* __restrict__ brp,
                                                 const uint64_t* __restrict__ poff,
                                                 const uint64_t* __restrict__ gpat, uint32_t* __restrict__ ac,
                                                 uint64_t* __restrict__ sp, uint8_t* __restrict__ packed,
                                                 const uint32_t* __restrict__ midlist,
                                                 const uint32_t* __restrict__ nmid,
                                                 uint32_t* __restrict__ hublist, uint32_t* __restrict__ hubch,
                                                 unsigned long long* __restrict__ nhub, uint32_t* work,
                                                 int hubs_done) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_scan[kEmitNT / 32 + 1];
  __shared__ uint32_t s_tt;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const int cap_blk = kSmallCap / tk + 1;
  unsigned long long* s_pt = reinterpret_cast<unsigned long long*>(dsm);       // [cap_blk * nbk] patterns
  uint64_t* s_vb = reinterpret_cast<uint64_t*>(s_pt + (size_t)cap_blk * nbk);  // [cap_blk] value base (bytes)
  uint16_t* s_so = reinterpret_cast<uint16_t*>(s_vb + cap_blk);                 // [cap_blk * nbk] value offsets
  uint8_t* s_row = reinterpret_cast<uint8_t*>(s_so + (size_t)cap_blk * nbk);    // [kSmallCap] row map
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t count = *nmid;
  while (true) {
    if (tid == 0) s_tt = atomicAdd(work, 1u);
    __syncthreads();
    const uint32_t tt = s_tt;
    if (tt >= count) break;
    const int64_t p = midlist[tt];
    const uint32_t b0 = brp[p], nblk = brp[p + 1] - b0;
    if (nblk == 0) {
      __syncthreads();
      continue;
    }
    const uint32_t nact = nact_in[p];
    load_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = s_rp[0], e1 = s_rp[nrows];
    const uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
    const bool small = e1 - e0 <= kSmallCap;  // (CTA-uniform; then nblk <= cap_blk)
    if (!small && hubs_done) continue;        // (k_count_hub + k_emit_hub own the hub panels)
    if (small) {
      for (int i = tid; i < (int)nblk * nbk; i += kEmitNT) s_pt[i] = gp[i];
      for (int r = warp; r < nrows; r += kEmitNT / 32) {
        const int b = (int)(s_rp[r] - e0), e = (int)(s_rp[r + 1] - e0);
        for (int i = b + lane; i < e; i += 32) s_row[i] = (uint8_t)r;
      }
      __syncthreads();
    }
    // blocks: sizes, sizePtr, headers, patterns, padding (chunks of kEmitNT blocks)
    uint64_t carry = poff[p];
    for (uint32_t c0 = 0; c0 < nblk; c0 += kEmitNT) {
      const uint32_t j = c0 + tid;
      uint32_t nbr = 0, nz = 0, size = 0;
      if (j < nblk) {
        for (int i = 0; i < nbk; ++i) {
          const uint64_t v = small ? s_pt[j * nbk + i] : gp[(int64_t)j * nbk + i];
          if (small) s_so[j * nbk + i] = (uint16_t)nz;  // values of the earlier bricks of the block (CSC order)
          nbr += v != 0ull;
          nz += __popcll(v);
        }
        size = block_bytes(nbc, nbr, nz);
      }
      uint32_t tot;
      const uint32_t ex = block_excl_scan<kEmitNT>(size, &tot, s_scan);
      if (j < nblk) {
        const uint64_t off = carry + ex;
        sp[b0 + j] = off;
        const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
        if (small) {
          s_vb[j] = off + hdr + 8 * nbr;
          if (nbc == 4 && nbrow == 1) {
            emit_block_meta<4, 1>(packed + off, s_pt + j * nbk, nbr, nz, size);
          } else {
            emit_block_meta_dyn(packed + off, s_pt + j * nbk, nbc, nbrow, nbr, nz, size);
          }
        } else {
          emit_block_meta_dyn(packed + off, reinterpret_cast<const unsigned long long*>(gp) + (int64_t)j * nbk, nbc,
                              nbrow, nbr, nz, size);
        }
      }
      carry += tot;
    }
    for (int64_t t = nact + tid; t < (int64_t)nblk * tk; t += kEmitNT) ac[(int64_t)b0 * tk + t] = (uint32_t)K;
    __syncthreads();  // sizePtr entries / staged metadata of this panel are visible to the whole CTA
    if (e1 - e0 > kHubEmit) {  // a hub's values are spread over every CTA by k_emit_hubvals (critical path)
      if (tid == 0) {  // one 64-bit atomic: (hub count << 32 | chunk count), so chunk bases rise with t
        const unsigned long long nch = (unsigned long long)((e1 - e0 + kHubChunk - 1) / kHubChunk);
        const unsigned long long old = atomicAdd(nhub, (1ull << 32) + nch);
        hublist[old >> 32] = (uint32_t)p;
        hubch[old >> 32] = (uint32_t)old;
      }
      continue;
    }
    if (small) {
      const int E = (int)(e1 - e0);
      for (int i = tid; i < E; i += kEmitNT) {  // values at popcount ranks, activeCols
        const uint32_t qq = q[e0 + i];
        const int32_t c = ci[e0 + i];
        const float v = vals[e0 + i];
        if (qq >= nact) continue;  // only for invalid CSR input
        const int r = s_row[i];
        const uint32_t j = qq / tk, lc = qq % tk;
        ac[((int64_t)b0 + j) * tk + lc] = (uint32_t)c;
        const int bit = ((r & 15) << 2) | (lc & 3);
        const int slot = (int)j * nbk + (lc >> 2) * nbrow + (r >> 4);
        const uint32_t off = s_so[slot] + __popcll(s_pt[slot] & ((1ull << bit) - 1ull));
        reinterpret_cast<float*>(packed + s_vb[j])[off] = v;
      }
      continue;
    }
    for (int64_t e = e0 + tid; e < e1; e += kEmitNT) {  // mid-size hubs: metadata from global memory
      const uint32_t qq = q[e];
      const int32_t c = ci[e];
      const float v = vals[e];
      if (qq >= nact) continue;  // only for invalid CSR input
      const int r = row_of(s_rp, nrows, e);
      const uint32_t j = qq / tk, lc = qq % tk;
      ac[((int64_t)b0 + j) * tk + lc] = (uint32_t)c;
      const int bit = ((r & 15) << 2) | (lc & 3);
      const int mine = (lc >> 2) * nbrow + (r >> 4);
      const uint64_t* pt = gp + (int64_t)j * nbk;
      uint32_t nbr = 0, off = 0;
      for (int i = 0; i < nbk; ++i) {
        const uint64_t w = pt[i];
        nbr += w != 0ull;
        if (i < mine) off += __popcll(w);
      }
      off += __popcll(pt[mine] & ((1ull << bit) - 1ull));
      const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
      reinterpret_cast<float*>(packed + sp[b0 + j] + hdr + 8 * nbr)[off] = v;
    }
  }  // panel loop
}

// Values + activeCols of hub panels (more than kHubEmit entries; R-MAT has panels of 600K entries, which one CTA
// took ~10 ms to scatter): every CTA takes a strided share of each hub's 4096-entry chunks. Block byte offsets,
// headers and patterns were written by k_emit; ranks q and patterns come from the count kernels' scratch.
__global__ void __launch_bounds__(kEmitThreads) k_emit_hubvals(const int64_t* __restrict__ rp,
                                                              const int32_t* __restrict__ ci,
                                                              const float* __restrict__ vals, int64_t M,
                                                              int64_t nnz, int tm, int tk,
                                                              const uint32_t* __restrict__ q,
                                                              const uint32_t* __restrict__ nact_in,
                                                              const uint32_t* __restrict__ brp,
                                                              const uint64_t* __restrict__ gpat,
                                                              uint32_t* __restrict__ ac, const uint64_t* __restrict__ sp,
                                                              uint8_t* __restrict__ packed,
                                                              const uint32_t* __restrict__ hublist,
                                                              const uint32_t* __restrict__ hubch,
                                                              const unsigned long long* __restrict__ nhub) {
  pdl_wait();
  __shared__ int64_t s_rp[129];
  const unsigned long long hc = *nhub;
  const uint32_t count = (uint32_t)(hc >> 32), total = (uint32_t)hc;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  for (uint32_t g = blockIdx.x; g < total; g += gridDim.x) {  // one flat list of every hub's chunks
    uint32_t lo = 0, hi = count - 1;  // last t with hubch[t] <= g
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (hubch[mid] <= g) lo = mid; else hi = mid - 1;
    }
    const int64_t p = hublist[lo];
    const int64_t ch = g - hubch[lo];
    load_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);  // (contains the barriers)
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = s_rp[0], e1 = s_rp[nrows];
    const uint32_t b0 = brp[p], nact = nact_in[p];
    const uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
    {
      const int64_t ce1 = min(e1, e0 + (ch + 1) * kHubChunk);
      for (int64_t e = e0 + ch * kHubChunk + threadIdx.x; e < ce1; e += blockDim.x) {
        const uint32_t qq = q[e];
        if (qq >= nact) continue;  // only for invalid CSR input
        const int r = row_of(s_rp, nrows, e);
        const uint32_t j = qq / tk, lc = qq % tk;
        ac[((int64_t)b0 + j) * tk + lc] = (uint32_t)ci[e];
        const int bit = ((r & 15) << 2) | (lc & 3);
        const int mine = (lc >> 2) * nbrow + (r >> 4);
        const uint64_t* pt = gp + (int64_t)j * nbk;
        uint32_t nbr = 0, off = 0;
        for (int i = 0; i < nbk; ++i) {
          const uint64_t w = pt[i];
          nbr += w != 0ull;
          if (i < mine) off += __popcll(w);
        }
        off += __popcll(pt[mine] & ((1ull << bit) - 1ull));
        const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
        reinterpret_cast<float*>(packed + sp[b0 + j] + hdr + 8 * nbr)[off] = vals[e];
      }
    }
  }
}

// status bits of asynchronous builds (graph replays of hrpb_build_spmm_async), ORed until read by
// hrpb_sync_status / the next synchronous replay (sticky_take)
__device__ unsigned int g_sticky_status;

__global__ void k_finalize(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int64_t P,
                           const uint32_t* __restrict__ brp, const uint64_t* __restrict__ poff,
                           uint64_t* __restrict__ sp, const uint32_t* __restrict__ status,
                           uint64_t* __restrict__ info, unsigned int* sticky) {
  pdl_wait();
  uint32_t st = *status;
  if (rp[0] != 0) st |= ST_RP0;
  if (rp[M] != nnz) st |= ST_NNZ;
  if (sticky && st) atomicOr(sticky, st);
  const uint64_t nb = brp[P];
  sp[nb] = poff[P];
  info[0] = nb;
  info[1] = poff[P];
  info[2] = st;
}

// ------------------------------------------------------------------ host orchestration
// warp-path kernels are specialised on (TM, TK) (compile-time brick-slot loops)
#define HRPB_WDISPATCH(CALL)                                                         \
  do {                                                                               \
    if (tk == 16) {                                                                  \
      if (tm == 16) { CALL(16, 16); } else if (tm == 32) { CALL(32, 16); }           \
      else if (tm == 64) { CALL(64, 16); } else { CALL(128, 16); }                   \
    } else {                                                                         \
      if (tm == 16) { CALL(16, 32); } else if (tm == 32) { CALL(32, 32); }           \
      else if (tm == 64) { CALL(64, 32); } else { CALL(128, 32); }                   \
    }                                                                                \
  } while (0)

template <int TM, int TK, int MODE>
static int wbuild_ctas() {  // resident CTAs of k_wbuild per SM (the ticket loop is persistent)
  static std::atomic<uint64_t> done{0};  // the shared-memory attribute is per device
  static std::atomic<int> n{0};
  if (first_on_device(done)) {
    const size_t smem = (size_t)warp_layout(TM, TK).bytes * kWWarps;
    cudaFuncSetAttribute(k_wbuild<TM, TK, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int m = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&m, k_wbuild<TM, TK, MODE>, 32 * kWWarps, smem);
    n = m < 1 ? 1 : m;
  }
  return n;
}
static void launch_wclassify(int tm, int tk, unsigned grid, cudaStream_t s, const int64_t* rp, const int32_t* ci,
                             int64_t M, int64_t nnz, int64_t P, uint8_t* listed, uint32_t* list, uint32_t* nlist,
                             uint32_t* biglist, uint32_t* nbig, uint32_t* nhuge, int64_t huge_cap) {
#define HRPB_WC(A, B) \
  k_wclassify<A, B><<<grid, 32 * kWWarps, 0, s>>>(rp, ci, M, nnz, P, listed, list, nlist, biglist, nbig, nhuge, huge_cap)
  HRPB_WDISPATCH(HRPB_WC);
#undef HRPB_WC
}

static void launch_wbuild(int mode, int tm, int tk, cudaStream_t s, const int64_t* rp, const int32_t* ci,
                          const float* vals, int64_t M, int64_t K, int64_t nnz, int64_t P, const uint8_t* listed,
                          const uint32_t* nblk_listed, const uint32_t* pbytes_listed, uint32_t* ticket,
                          uint64_t* lb, uint32_t* brp, uint64_t* poff, uint32_t* ac,
                          uint64_t* sp, uint8_t* packed, uint32_t* status) {
  const size_t smem = (size_t)warp_layout(tm, tk).bytes * kWWarps;
#define HRPB_WB_M(A, B, MO)                                                                                    \
  {                                                                                                            \
    const int64_t want = ceil_div(P, kWWarps), have = (int64_t)wbuild_ctas<A, B, MO>() * num_sms();            \
    launch_pdl(k_wbuild<A, B, MO>, (unsigned)(want < have ? want : have), 32 * kWWarps, smem, s,               \
        rp, ci, vals, M, K, nnz, P, listed, nblk_listed, pbytes_listed, ticket, lb, brp, poff,                \
        ac, sp, packed, status);                                                                               \
  }
#define HRPB_WB(A, B)                                                                                          \
  {                                                                                                            \
    if (mode == 1) HRPB_WB_M(A, B, 1) else if (mode == 2) HRPB_WB_M(A, B, 2) else HRPB_WB_M(A, B, 0)          \
  }
  HRPB_WDISPATCH(HRPB_WB);
#undef HRPB_WB
#undef HRPB_WB_M
}

// three-phase warp path (count, scan, emit) instead of the single pass with look-back: chosen by panel count
// (HRPB_WB_MODE=1 / 0 forces it on / off for experiments). Measured (build ms, single pass -> three-phase): c3
// (262K panels, 24% listed, warp panels of 1..512 entries) 5.69 -> 5.31; c4 (131K uniform 128-entry panels) 0.79
// -> 0.99; c2a / c2b (16K panels at TM = 64) 0.27 -> 0.34; c5 (31K listed panels) 1.10 -> 1.07. The look-back
// only costs when thousands of in-flight panels of very different sizes wait on each other, which takes a large
// panel count; the count pass repeats the ranking, which costs on uniform matrices.
static bool use_three_phase(int64_t M, int64_t nnz, int64_t P, int tm) {
  static const int forced = [] {
    const char* e = getenv("HRPB_WB_MODE");
    return e ? atoi(e) : -1;
  }();
  if (forced >= 0) return forced != 0;
  (void)M; (void)nnz; (void)tm;
  return P >= kThreePhaseMinPanels;
}

hrpb_status_t build_impl(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                         const float* values, int32_t tm, int32_t tk, cudaStream_t s, hrpb_handle* h,
                         uint64_t* deferred_info, bool sticky) {
  const int64_t P = ceil_div(M, tm);
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  // upper bounds (no host round trip): sum_p ceil(nact_p/tk) <= nnz/tk + min(P, nnz)
  const int64_t nb_cap = nnz / tk + (P < nnz ? P : nnz);
  const int64_t hdr_cap = align_up(nbc + 1 + nbk, 8) + 15;
  const int64_t brick_cap = nnz < nb_cap * nbk ? nnz : nb_cap * nbk;
  const int64_t bytes_cap = nb_cap * hdr_cap + 8 * brick_cap + 4 * nnz;
  const int64_t pat_cap = nnz * nbk / tk + 2 * (P + 1) * nbk + nbk;

  h->M = M; h->K = K; h->nnz = nnz; h->P = P; h->tm = tm; h->tk = tk; h->stream = s;
  h->brp = (uint32_t*)dalloc((P + 1) * sizeof(uint32_t), s);
  h->ac = (uint32_t*)dalloc((nb_cap * tk + 1) * sizeof(uint32_t), s);
  h->sp = (uint64_t*)dalloc((nb_cap + 1) * sizeof(uint64_t), s);
  h->packed = (uint8_t*)dalloc(bytes_cap + 16, s);
  uint32_t* q = (uint32_t*)dalloc((nnz + 1) * sizeof(uint32_t), s);
  uint32_t* cnt = (uint32_t*)dalloc(3 * (P + 1) * sizeof(uint32_t), s);  // nact | nblk | panel bytes
  uint32_t* nact = cnt;
  uint32_t* nblk = cnt + (P + 1);
  uint32_t* pbytes = cnt + 2 * (P + 1);
  uint64_t* poff = (uint64_t*)dalloc((P + 1) * sizeof(uint64_t), s);
  uint64_t* gpat = (uint64_t*)dalloc(pat_cap * sizeof(uint64_t), s);
  // panel lists: big (> kSmallCap entries, hub bitmap) | L1 (not on the warp path: CTA count + CTA emit)
  uint32_t* biglist = (uint32_t*)dalloc(3 * (P + 1) * sizeof(uint32_t), s);
  uint32_t* l1 = biglist + (P + 1);
  // nbig, nl1, ticket, hub work, status, emit work, hub (count << 32 | chunks) x2, count work
  uint32_t* ctr = (uint32_t*)dalloc(16 * sizeof(uint32_t), s);
  uint64_t* lb = (uint64_t*)dalloc((P + 1) * sizeof(uint64_t), s);  // look-back states (blocks << 34 | bytes)
  // three-phase warp path (see k_wbuild): when not every panel is on the warp path, or on many small panels
  const bool three_phase = use_three_phase(M, nnz, P, tm);
  uint64_t* lbx = nullptr;
  void* scan_tmp_p = nullptr;
  size_t scan_tmp = 0;
  if (three_phase && P > 0) {
    cub::DeviceScan::ExclusiveSum(nullptr, scan_tmp, lb, lb, (int)(P + 1), s);
    lbx = (uint64_t*)dalloc((P + 1) * sizeof(uint64_t) + scan_tmp + 16, s);
    scan_tmp_p = lbx ? (void*)(lbx + P + 1) : nullptr;
  }
  uint8_t* listed = (uint8_t*)dalloc(P + 1, s);
  uint64_t* info = (uint64_t*)dalloc(4 * sizeof(uint64_t), s);  // [3] = status word | hub count
  const int big_ctas = HRPB_BIG_CTAS_PER_SM * num_sms();
  const int64_t words = ceil_div(K, 32) + 2;
  // hub panels: dense shared-memory passes (k_count_hub / k_emit_hub) when the per-row pass boundaries fit, else
  // the global occupancy-bitmap kernel (k_count_big, with k_emit / k_emit_hubvals)
  static const bool force_old_hub = [] {
    const char* e = getenv("HRPB_HUB_GLOBAL");  // experiments: the global-bitmap hub path
    return e && atoi(e);
  }();
  const bool hub_2l = hub2_ok(K) && !force_old_hub;
  const bool hub_dense = (hub_2l || hub_dense_ok(K, tm)) && !force_old_hub;
  const int hub2_ctas = HRPB_H2_MINB * num_sms();
  uint32_t* bigscr = hub_2l ? (uint32_t*)dalloc((size_t)hub2_ctas * 2 * ceil_div(K, 32) * sizeof(uint32_t) + 16, s)
                     : hub_dense ? (uint32_t*)dalloc(16, s)
                                 : (uint32_t*)dalloc((size_t)big_ctas * (2 * words + 2 * ((words + 31) / 32)) *
                                                     sizeof(uint32_t), s);
  uint32_t* relb = (uint32_t*)dalloc((nnz / tk + 2 * P + 4) * sizeof(uint32_t), s);  // hub blocks' relative offsets
  uint32_t* hub2 = (uint32_t*)dalloc(2 * (P + 1) * sizeof(uint32_t), s);
  hrpb_status_t st = HRPB_SUCCESS;
  // the fused look-back packs (blocks, bytes) into 62 bits
  if (nb_cap >= (1ll << 28) || bytes_cap >= (1ll << 34)) {
    st = HRPB_ERROR_NOT_SUPPORTED;
  } else if (!h->brp || !h->ac || !h->sp || !h->packed || !q || !cnt || !poff || !gpat || !biglist || !info ||
             !bigscr || !ctr || !lb || !listed || !relb || !hub2 || (three_phase && P > 0 && !lbx)) {
    st = HRPB_ERROR_OUT_OF_MEMORY;
  }
  uint64_t hinfo[3] = {0, 0, 0};
  if (st == HRPB_SUCCESS) {
    uint32_t* nbig = ctr;
    uint32_t* nl1 = ctr + 1;
    uint32_t* ticket = ctr + 2;
    unsigned long long* nhub = reinterpret_cast<unsigned long long*>(ctr + 6);  // (hubs << 32 | chunks)
    uint32_t* hublist = biglist;  // (the big list is consumed by k_count_big before k_emit reuses it)
    uint32_t* hubch = biglist + 2 * (P + 1);
    // dense hub path: its own (hub, work-item prefix) list, written by k_count_hub while it still reads the big list
    uint32_t* hublist2 = hub2;
    uint32_t* hubch2 = hub2 + (P + 1);
    unsigned long long* nhub2 = reinterpret_cast<unsigned long long*>(ctr + 10);
    uint32_t* status = ctr + 4;
    cudaMemsetAsync(ctr, 0, 16 * sizeof(uint32_t), s);
    const size_t count_smem = mid_smem_bytes(tm, tk), emit_smem = emit_smem_bytes(tm, tk);
    static std::atomic<uint64_t> attr{0};  // per device
    if (first_on_device(attr)) {
      cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_emit, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_count_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(HubSmem));
      cudaFuncSetAttribute(k_count_hub2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Hub2Smem));
    }
    const unsigned wgrid = (unsigned)ceil_div(P, kWWarps);
    const int mid_ctas = 8 * num_sms();
    const int count_ctas = (int)(227 * 1024 / (count_smem + 1024)) * num_sms();
    const int emit_ctas = (int)min((size_t)(2048 / kEmitNT), 227 * 1024 / (emit_smem + 1024)) * num_sms();
    cudaMemsetAsync(lb, 0, (P + 1) * sizeof(uint64_t), s);
    cudaMemsetAsync(h->brp, 0, sizeof(uint32_t), s);  // P == 0: blockedRowPtr = {0}
    cudaMemsetAsync(poff, 0, sizeof(uint64_t), s);
    if (P > 0) {
      // classification: warp-path panels, listed panels (counted by a CTA, <= kSmallCap entries) and hub panels
      // (measured: running the hub kernels on a side stream beside the listed-panel kernels gained nothing on c3 —
      // each fills the SMs' shared memory, so they do not co-reside)
      const int64_t huge_cap = hub_2l ? kH2Huge : (int64_t)0;
      launch_wclassify(tm, tk, wgrid, s, row_ptr, col_idx, M, nnz, P, listed, l1, nl1, biglist, nbig, ctr + 12,
                       huge_cap);
      launch_pdl(k_count, count_ctas, kMidThreads, count_smem, s, row_ptr, col_idx, M, K, nnz, tm, tk, q, nact, nblk,
                 pbytes, gpat, l1, nl1, biglist, nbig, ctr + 8, status, ctr + 12, huge_cap, P);
      if (hub_2l)
        launch_pdl(k_count_hub2, hub2_ctas, kH2Threads, sizeof(Hub2Smem), s, row_ptr, col_idx, M, K, nnz, tm, tk, q,
                   nact, nblk, pbytes, gpat, relb, biglist, nbig, ctr + 3, hublist2, hubch2, nhub2, bigscr, status,
                   ctr + 12, P);
      else if (hub_dense)
        launch_pdl(k_count_hub, num_sms(), kHubThreads, sizeof(HubSmem), s, row_ptr, col_idx, M, K, nnz, tm, tk, q,
                   nact, nblk, pbytes, gpat, relb, biglist, nbig, ctr + 3, hublist2, hubch2, nhub2, status);
      else
        launch_pdl(k_count_big, big_ctas, kBigThreads, 0, s, row_ptr, col_idx, M, K, nnz, tm, tk, q, nact, nblk,
                   pbytes, gpat, biglist, nbig, bigscr, words, ctr + 3, status);
      // B1-B5 for warp-path panels + the scans B2 / B4 for all panels: one pass with a decoupled look-back, or
      // (three-phase) count pass, device scan of the packed (blocks << 34 | bytes), emit pass
      if (three_phase) {
        launch_wbuild(1, tm, tk, s, row_ptr, col_idx, values, M, K, nnz, P, listed, nblk, pbytes, ctr + 14, lb,
                      h->brp, poff, h->ac, h->sp, h->packed, status);
        size_t tb = scan_tmp;
        cub::DeviceScan::ExclusiveSum(scan_tmp_p, tb, lb, lbx, (int)(P + 1), s);
        launch_wbuild(2, tm, tk, s, row_ptr, col_idx, values, M, K, nnz, P, listed, nblk, pbytes, ticket, lbx,
                      h->brp, poff, h->ac, h->sp, h->packed, status);
        note_launch(1);  // the second k_wbuild (the CUB scan kernels are library code, not counted)
      } else {
        launch_wbuild(0, tm, tk, s, row_ptr, col_idx, values, M, K, nnz, P, listed, nblk, pbytes, ticket, lb,
                      h->brp, poff, h->ac, h->sp, h->packed, status);
      }
      launch_pdl(k_emit, emit_ctas, kEmitNT, emit_smem, s, row_ptr, col_idx, values, M, K, nnz, tm, tk, q, nact, h->brp,
                 poff, gpat, h->ac, h->sp, h->packed, l1, nl1, hublist, hubch, nhub, ctr + 5, (int)hub_dense);
      if (hub_2l)
        launch_pdl(k_emit_hub2, kE2MinB * num_sms(), kE2Threads, 0, s, row_ptr, col_idx, values, M, K, nnz, tm, tk, q, nact,
                   h->brp, poff, gpat, relb, h->ac, h->sp, h->packed, hublist2, hubch2, nhub2);
      else if (hub_dense)
        launch_pdl(k_emit_hub, mid_ctas, kEmitHubNT, 0, s, row_ptr, col_idx, values, M, K, nnz, tm, tk, q, nact, h->brp,
                   poff, gpat, relb, h->ac, h->sp, h->packed, hublist2, hubch2, nhub2);
      else
        launch_pdl(k_emit_hubvals, mid_ctas, kEmitThreads, 0, s, row_ptr, col_idx, values, M, nnz, tm, tk, q, nact,
                   h->brp, gpat, h->ac, h->sp, h->packed, hublist, hubch, nhub);
      note_launch(6);
    }
    unsigned int* sticky_p = nullptr;
    if (sticky) cudaGetSymbolAddress(reinterpret_cast<void**>(&sticky_p), g_sticky_status);
    launch_pdl(k_finalize, 1, 1, 0, s, row_ptr, M, nnz, P, h->brp, poff, h->sp, status, info, sticky_p);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (deferred_info) {  // (NUM_BLKS, bytes, status) land in the caller's pinned buffer; it syncs and finishes
      if (e == cudaSuccess) e = cudaMemcpyAsync(deferred_info, info, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    } else {
      if (e == cudaSuccess) e = cudaMemcpyAsync(hinfo, info, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    }
    if (e != cudaSuccess) st = cuda_status(e);
#ifdef HRPB_BTRACE
    unsigned long long bt[8];
    cudaMemcpyFromSymbol(bt, g_btrace, sizeof(bt));
    fprintf(stderr, "btrace cycles (sum over warps): ticket %.3g rows %.3g stage %.3g rank %.3g patterns %.3g "
            "lookback %.3g emit %.3g\n", (double)bt[0], (double)bt[1], (double)bt[2], (double)bt[3], (double)bt[4],
            (double)bt[5], (double)bt[6]);
    const unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbol(g_btrace, z, sizeof(z));
    unsigned long long ls[4];
    cudaMemcpyFromSymbol(ls, g_lbstat, sizeof(ls));
    fprintf(stderr, "look-back: %llu panels, %.2f load rounds and %.2f polls per panel\n", ls[0],
            (double)ls[1] / (double)(ls[0] ? ls[0] : 1), (double)ls[2] / (double)(ls[0] ? ls[0] : 1));
    cudaMemcpyToSymbol(g_lbstat, z, sizeof(ls));
#endif
  }
  dfree(q, s); dfree(cnt, s); dfree(poff, s); dfree(gpat, s); dfree(biglist, s); dfree(info, s);
  dfree(bigscr, s); dfree(relb, s); dfree(hub2, s);
  dfree(ctr, s); dfree(lb, s); dfree(lbx, s); dfree(listed, s);
  if (deferred_info) {
    h->NB = -1;  // unknown until build_finish
    return st;
  }
  return build_finish(h, hinfo, st);
}

// read-and-clear of the sticky status word in one atomic (a replay on another stream that ORs its status in
// between a separate read and clear would otherwise be lost)
__global__ void k_sticky_take(unsigned int* sticky, unsigned int* out) { *out = atomicExch(sticky, 0u); }

hrpb_status_t sticky_take(cudaStream_t s) {
  unsigned int* addr = nullptr;
  cudaError_t e = cudaGetSymbolAddress(reinterpret_cast<void**>(&addr), g_sticky_status);
  unsigned int* word = (unsigned int*)dalloc(sizeof(unsigned int), s);
  if (!word) return HRPB_ERROR_OUT_OF_MEMORY;
  unsigned int v = 0;
  if (e == cudaSuccess) {
    k_sticky_take<<<1, 1, 0, s>>>(addr, word);
    note_launch();
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(&v, word, sizeof(v), cudaMemcpyDeviceToHost, s);
  dfree(word, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e);
  return v ? HRPB_ERROR_INVALID_CSR : HRPB_SUCCESS;
}

// ------------------------------------------------------------------ automatic TM (hrpb_config_t.tm = 0)
// NEXT-1 ("TM either 16 or 32"; the beta reuse of P:L329-357): taller panels share gathered B rows between
// more output rows but multiply zero-filled brick rows. The choice is made from B1 statistics of a sample: up to
// kProbeSamples evenly spaced 64-row groups, each ranked as one TM = 64 panel and as four TM = 16 panels
// (CTA radix sort of (column, sub-panel) keys, distinct columns counted per sub-panel and overall). Groups with
// more than kProbeCap entries count as TM-neutral (their blocks at either TM ~ entries / TK).
constexpr int kProbeThreads = 256, kProbeItems = 8, kProbeCap = kProbeThreads * kProbeItems;
constexpr int64_t kProbeSamples = 1024;

__global__ void __launch_bounds__(kProbeThreads) k_tm_probe(const int64_t* __restrict__ rp,
                                                            const int32_t* __restrict__ ci, int64_t M, int64_t nnz,
                                                            int64_t groups, int64_t samples, int key_bits,
                                                            unsigned long long* __restrict__ acc) {
  pdl_wait();
  using Sort = cub::BlockRadixSort<unsigned long long, kProbeThreads, kProbeItems>;
  __shared__ typename Sort::TempStorage tmp;
  __shared__ unsigned long long s_keys[kProbeCap];
  __shared__ int64_t s_rp[65];
  __shared__ uint32_t s_cnt[5];  // distinct columns of the 64-row group, then of each 16-row sub-panel
  for (int64_t i = blockIdx.x; i < samples; i += gridDim.x) {
    const int64_t g = i * groups / samples;
    const int64_t r0 = g * 64;
    const int nrows = (int)min((int64_t)64, M - r0);
    __syncthreads();
    if (threadIdx.x <= nrows) {
      const int64_t v = rp[r0 + threadIdx.x];
      s_rp[threadIdx.x] = v < 0 ? 0 : (v > nnz ? nnz : v);
    }
    if (threadIdx.x < 5) s_cnt[threadIdx.x] = 0u;
    __syncthreads();
    const int64_t e0 = s_rp[0];
    const int64_t E = s_rp[nrows] - e0;
    if (E <= 0) continue;  // (CTA-uniform)
    const int nsub = (nrows + 15) / 16;
    if (E > kProbeCap) {
      if (threadIdx.x == 0) {
        const unsigned long long nb = (unsigned long long)((E + 15) / 16);
        atomicAdd(&acc[0], nb);
        atomicAdd(&acc[1], nb);
        atomicAdd(&acc[2], (unsigned long long)nsub);
      }
      continue;
    }
    unsigned long long key[kProbeItems];
#pragma unroll
    for (int k = 0; k < kProbeItems; ++k) {
      const int idx = threadIdx.x * kProbeItems + k;
      key[k] = ~0ull;
      if (idx < E) {
        int lo = 0, hi = nrows - 1;  // local row of entry idx
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_rp[mid] - e0 <= idx) lo = mid; else hi = mid - 1;
        }
        const int32_t c = ci[e0 + idx];
        key[k] = ((unsigned long long)(uint32_t)max(c, 0) << 2) | (unsigned long long)(lo >> 4);
      }
    }
    Sort(tmp).Sort(key, 0, key_bits);
#pragma unroll
    for (int k = 0; k < kProbeItems; ++k) s_keys[threadIdx.x * kProbeItems + k] = key[k];
    __syncthreads();
    uint32_t n64 = 0, n16[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < kProbeItems; ++k) {
      const int idx = threadIdx.x * kProbeItems + k;
      if (idx >= E) continue;
      const unsigned long long cur = key[k], prev = idx ? s_keys[idx - 1] : ~0ull;
      if (idx == 0 || (cur >> 2) != (prev >> 2)) ++n64;
      if (idx == 0 || cur != prev) ++n16[cur & 3];
    }
    if (n64) atomicAdd(&s_cnt[0], n64);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (n16[k]) atomicAdd(&s_cnt[1 + k], n16[k]);
    __syncthreads();
    if (threadIdx.x == 0) {
      unsigned long long nb16 = 0;
      for (int k = 0; k < 4; ++k) nb16 += (s_cnt[1 + k] + 15) / 16;
      atomicAdd(&acc[0], nb16);
      atomicAdd(&acc[1], (unsigned long long)((s_cnt[0] + 15) / 16));
      atomicAdd(&acc[2], (unsigned long long)nsub);
    }
  }
}

hrpb_status_t choose_tm(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                        cudaStream_t s, int32_t* tm_out, uint64_t* stats) {
  *tm_out = 16;
  const int64_t groups = ceil_div(M, 64);
  if (groups == 0 || nnz == 0) return HRPB_SUCCESS;
  unsigned long long* acc = (unsigned long long*)dalloc(4 * sizeof(unsigned long long), s);
  if (!acc) return HRPB_ERROR_OUT_OF_MEMORY;
  unsigned long long h[4] = {0, 0, 0, 0};
  cudaError_t e = cudaMemsetAsync(acc, 0, 4 * sizeof(unsigned long long), s);
  const int64_t samples = groups < kProbeSamples ? groups : kProbeSamples;
  int kb = 2;
  while (kb < 64 && (1ll << (kb - 2)) < K) ++kb;
  if (e == cudaSuccess) {
    const unsigned grid = (unsigned)(samples < 2 * num_sms() ? samples : 2 * num_sms());
    e = launch_pdl(k_tm_probe, grid, kProbeThreads, 0, s, row_ptr, col_idx, M, nnz, groups, samples, kb, acc);
    note_launch();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(h, acc, sizeof(h), cudaMemcpyDeviceToHost, s);
  dfree(acc, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return cuda_status(e);
  if (stats) { stats[0] = h[0]; stats[1] = h[1]; stats[2] = h[2]; }
  // Measured on B200 (profiles/r01/configs.md, DESIGN.md NEXT-1): the SpMM is bound by per-block work at both TM
  // (a TM = 64 block costs ~1.5x a TM = 16 block), so TM = 64 pays when it cuts the blocks to < 2/3 (c2a: 0.40),
  // or when TM = 16 panels hold about one block each, whose per-panel epilogue then dominates (c2b: 1.0 block per
  // panel, 0.99 of the blocks). Otherwise (c1, c3, c4, c5: 0.68-1.0 of the blocks, 7-28 blocks per panel) TM = 16.
  if (h[0] > 0) {
    const double r = (double)h[1] / (double)h[0], bpp = (double)h[0] / (double)(h[2] ? h[2] : 1);
    if (r < 0.67 || (bpp <= 1.5 && r <= 1.05)) *tm_out = 64;
  }
  return HRPB_SUCCESS;
}

hrpb_status_t build_finish(hrpb_handle* h, const uint64_t* info, hrpb_status_t st) {
  if (st == HRPB_SUCCESS && info[2] != 0) st = HRPB_ERROR_INVALID_CSR;
  h->NB = (int64_t)info[0];
  h->bytes = (int64_t)info[1];
  return st;
}

}  // namespace hrpb
