// build.cu — GPU CSR -> HRPB builder, bit-identical to the oracle.
//
// Paper: Alg. "CSR to HRPB Phase1/Phase2" runs on the host with OpenMP over panel
// chunks and prefix sums; §"HRPB Sparse Matrix Data structure" defines the output.
// B200 design: no host round trip until the end; outputs are allocated at
// upper bounds computable from (M, nnz), so the pipeline is
//   k_rank_small / k_rank_big  (B1: per-panel sorted-unique active columns -> compacted rank q of
//                               every entry, nact per panel; validation of the CSR)
//   scan(nblk) -> blockedRowPtr (B2)
//   k_fill                     (B3: activeCols incl. sentinel K, brick patterns, block sizes)
//   scan(size) -> sizePtr      (B4)
//   k_pack                     (B5: HRPB-v1 headers, patterns, values in brick-CSC / row-major order)
//   k_finalize                 (NUM_BLKS, byte total, status) -> one 32-byte D2H read + sync.
#include <cstdio>

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
constexpr int kSmallCap = 2048;      // entries per panel handled in shared memory (bitonic path)
constexpr int kSpanWords = 512;      // bitmap path when the panel's column span <= 16384
constexpr int kBigThreads = 512;
constexpr int kFillThreads = 128;
constexpr int kFillSmemBricks = 1024;  // patterns kept in shared memory up to this many bricks

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

struct PanelRows {
  int64_t r0, r1;  // rows [r0, r1)
};

// Loads the (clamped, monotone-repaired) row pointers of panel p into shared memory; thread 0 flags a
// decreasing row_ptr in *status (if non-null). Clamping keeps every later access inside [0, nnz).
__device__ __forceinline__ void load_panel_rows(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int tm,
                                                int64_t p, int64_t* s_rp, uint32_t* status) {
  const int64_t r0 = p * tm;
  const int nrows = (int)min((int64_t)tm, M - r0);
  __syncthreads();
  for (int i = threadIdx.x; i <= nrows; i += blockDim.x) {
    int64_t v = rp[r0 + i];
    s_rp[i] = v < 0 ? 0 : (v > nnz ? nnz : v);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    bool bad = false;
    for (int i = 1; i <= nrows; ++i) {
      if (rp[r0 + i] < rp[r0 + i - 1]) bad = true;
      if (s_rp[i] < s_rp[i - 1]) s_rp[i] = s_rp[i - 1];
    }
    if (bad && status) atomicOr(status, ST_RP_MONO);
  }
  __syncthreads();
}

// ------------------------------------------------------------------ B1: panels with <= kSmallCap entries
// One CTA per panel. q[e] = rank of col_idx[e] among the panel's distinct columns (ascending, R23),
// nact[p] = number of distinct columns ("active_cols = uniq(cols[row_start: row_end])").
__global__ void __launch_bounds__(kSmallThreads) k_rank_small(const int64_t* __restrict__ rp,
                                                             const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                             int64_t nnz, int tm, int tk, uint32_t* __restrict__ q,
                                                             uint32_t* __restrict__ nact_out,
                                                             uint32_t* __restrict__ nblk_out, uint32_t* status) {
  __shared__ int64_t s_rp[129];
  __shared__ __align__(16) uint64_t s_keys[kSmallCap];  // also reused as the bitmap (2 x 512 words)
  __shared__ uint32_t s_scan[kSmallThreads / 32 + 1];
  __shared__ int32_t s_mm[2 * kSmallThreads / 32];
  const int64_t p = blockIdx.x;
  load_panel_rows(rp, M, nnz, tm, p, s_rp, status);
  const int nrows = (int)min((int64_t)tm, M - p * tm);
  const int64_t e0 = s_rp[0];
  const int64_t E = s_rp[nrows] - e0;
  if (E > kSmallCap) return;  // handled by k_rank_big (uniform exit: E is CTA-uniform)
  if (E == 0) {
    if (threadIdx.x == 0) { nact_out[p] = 0; nblk_out[p] = 0; }
    return;
  }
  // validation + column span
  int32_t mn = INT32_MAX, mx = INT32_MIN;
  for (int r = 0; r < nrows; ++r) {
    for (int64_t e = s_rp[r] + threadIdx.x; e < s_rp[r + 1]; e += blockDim.x) {
      int32_t c = ci[e];
      if (c < 0 || c >= K) atomicOr(status, ST_COL_RANGE);
      if (e > s_rp[r] && ci[e - 1] >= c) atomicOr(status, ST_COL_ORDER);
      mn = min(mn, c);
      mx = max(mx, c);
    }
  }
  block_minmax<kSmallThreads>(mn, mx, s_mm);
  uint32_t nact = 0;
  const int64_t span = (int64_t)mx - (int64_t)mn + 1;
  if (span <= 32 * kSpanWords) {
    // bitmap path: set bits, popcount prefix per word, rank = prefix + popc(word & below)
    uint32_t* bm = reinterpret_cast<uint32_t*>(s_keys);
    uint32_t* pre = bm + kSpanWords;
    for (int i = threadIdx.x; i < kSpanWords; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e0 + E; e += blockDim.x) {
      uint32_t off = (uint32_t)(ci[e] - mn);
      atomicOr(&bm[off >> 5], 1u << (off & 31));
    }
    __syncthreads();
    constexpr int kPer = kSpanWords / kSmallThreads;
    uint32_t cnt[kPer], sum = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) { cnt[i] = __popc(bm[threadIdx.x * kPer + i]); sum += cnt[i]; }
    uint32_t run = block_excl_scan<kSmallThreads>(sum, &nact, s_scan);
#pragma unroll
    for (int i = 0; i < kPer; ++i) { pre[threadIdx.x * kPer + i] = run; run += cnt[i]; }
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e0 + E; e += blockDim.x) {
      uint32_t off = (uint32_t)(ci[e] - mn);
      uint32_t w = off >> 5, b = off & 31;
      q[e] = pre[w] + __popc(bm[w] & ((1u << b) - 1u));
    }
  } else {
    // sort path: bitonic sort of (col << 32 | local index), then unique ranks
    int n = 32;
    while (n < E) n <<= 1;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      s_keys[i] = i < E ? ((uint64_t)(uint32_t)ci[e0 + i] << 32) | (uint32_t)i : ~0ull;
    __syncthreads();
    for (int k = 2; k <= n; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          int ixj = i ^ j;
          if (ixj > i) {
            uint64_t a = s_keys[i], b = s_keys[ixj];
            bool up = (i & k) == 0;
            if ((a > b) == up) { s_keys[i] = b; s_keys[ixj] = a; }
          }
        }
        __syncthreads();
      }
    }
    // ranks: chunk of consecutive sorted positions per thread
    const int per = n / kSmallThreads > 0 ? n / kSmallThreads : 1;
    const int beg = threadIdx.x * per;
    uint32_t sum = 0;
    for (int i = beg; i < beg + per && i < n; ++i)
      if (i < E && (i == 0 || (s_keys[i] >> 32) != (s_keys[i - 1] >> 32))) ++sum;
    uint32_t run = block_excl_scan<kSmallThreads>(sum, &nact, s_scan);
    for (int i = beg; i < beg + per && i < n; ++i) {
      if (i >= E) break;
      if (i == 0 || (s_keys[i] >> 32) != (s_keys[i - 1] >> 32)) ++run;
      q[e0 + (uint32_t)s_keys[i]] = run - 1;
    }
  }
  if (threadIdx.x == 0) {
    nact_out[p] = nact;
    nblk_out[p] = (nact + tk - 1) / tk;  // reading R1: ceil(nact / TK)
  }
}

// ------------------------------------------------------------------ B1: panels with > kSmallCap entries
// Persistent CTAs; each owns a global bitmap over the panel's column span (words + prefix).
__global__ void __launch_bounds__(kBigThreads) k_rank_big(const int64_t* __restrict__ rp,
                                                         const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                         int64_t nnz, int tm, int tk, int64_t P,
                                                         uint32_t* __restrict__ q, uint32_t* __restrict__ nact_out,
                                                         uint32_t* __restrict__ nblk_out, uint32_t* scratch,
                                                         int64_t words_per_cta, uint32_t* status) {
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_scan[kBigThreads / 32 + 1];
  __shared__ int32_t s_mm[2 * kBigThreads / 32];
  uint32_t* bm = scratch + (int64_t)blockIdx.x * 2 * words_per_cta;
  uint32_t* pre = bm + words_per_cta;
  for (int64_t p = blockIdx.x; p < P; p += gridDim.x) {
    int64_t r0 = p * tm;
    int nrows = (int)min((int64_t)tm, M - r0);
    int64_t a = rp[r0], b = rp[r0 + nrows];
    a = a < 0 ? 0 : (a > nnz ? nnz : a);
    b = b < 0 ? 0 : (b > nnz ? nnz : b);
    if (b - a <= kSmallCap) continue;  // CTA-uniform
    __syncthreads();
    load_panel_rows(rp, M, nnz, tm, p, s_rp, status);
    const int64_t e0 = s_rp[0], e1 = s_rp[nrows];
    int32_t mn = INT32_MAX, mx = INT32_MIN;
    for (int r = 0; r < nrows; ++r) {
      for (int64_t e = s_rp[r] + threadIdx.x; e < s_rp[r + 1]; e += blockDim.x) {
        int32_t c = ci[e];
        bool ok = c >= 0 && c < K;
        if (!ok) atomicOr(status, ST_COL_RANGE);
        if (e > s_rp[r] && ci[e - 1] >= c) atomicOr(status, ST_COL_ORDER);
        if (ok) { mn = min(mn, c); mx = max(mx, c); }
      }
    }
    block_minmax<kBigThreads>(mn, mx, s_mm);
    if (mn > mx) { mn = 0; mx = 0; }
    const int64_t base = mn >> 5;
    const int64_t W = (mx >> 5) - base + 1;
    for (int64_t i = threadIdx.x; i < W; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      int32_t c = ci[e];
      if (c >= 0 && c < K) atomicOr(&bm[(c >> 5) - base], 1u << (c & 31));
    }
    __threadfence_block();
    __syncthreads();
    const int64_t per = (W + blockDim.x - 1) / blockDim.x;
    const int64_t beg = threadIdx.x * per, end = min(W, beg + per);
    uint32_t sum = 0;
    for (int64_t i = beg; i < end; ++i) sum += __popc(__ldcg(&bm[i]));
    uint32_t nact;
    uint32_t run = block_excl_scan<kBigThreads>(sum, &nact, s_scan);
    for (int64_t i = beg; i < end; ++i) { pre[i] = run; run += __popc(__ldcg(&bm[i])); }
    __threadfence_block();
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      int32_t c = ci[e];
      if (c < 0 || c >= K) { q[e] = 0xFFFFFFFFu; continue; }
      int64_t w = (c >> 5) - base;
      q[e] = __ldcg(&pre[w]) + __popc(__ldcg(&bm[w]) & ((1u << (c & 31)) - 1u));
    }
    if (threadIdx.x == 0) {
      nact_out[p] = nact;
      nblk_out[p] = (nact + tk - 1) / tk;
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------ device-wide exclusive scan
constexpr int kScanThreads = 256, kScanPer = 16, kScanChunk = kScanThreads * kScanPer;

__global__ void __launch_bounds__(kScanThreads) k_scan_partials(const uint32_t* __restrict__ in, int64_t n,
                                                                uint64_t* __restrict__ part) {
  __shared__ uint64_t sh[kScanThreads / 32];
  int64_t base = (int64_t)blockIdx.x * kScanChunk;
  uint64_t s = 0;
  for (int i = 0; i < kScanPer; ++i) {
    int64_t idx = base + (int64_t)i * kScanThreads + threadIdx.x;
    if (idx < n) s += in[idx];
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) t += sh[w];
    part[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(1024) k_scan_top(uint64_t* part, int64_t nparts) {
  __shared__ uint64_t sh[33];
  uint64_t carry = 0;
  for (int64_t base = 0; base < nparts; base += 1024) {
    int64_t i = base + threadIdx.x;
    uint64_t v = i < nparts ? part[i] : 0, x = v;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) sh[warp] = x;
    __syncthreads();
    if (warp == 0) {
      uint64_t w = sh[lane];
      for (int o = 1; o < 32; o <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      sh[lane] = w;
    }
    __syncthreads();
    uint64_t excl = carry + (warp ? sh[warp - 1] : 0) + x - v;
    uint64_t tot = sh[31];
    __syncthreads();
    if (i < nparts) part[i] = excl;
    carry += tot;
  }
}

template <typename OutT>
__global__ void __launch_bounds__(kScanThreads) k_scan_down(const uint32_t* __restrict__ in, int64_t n,
                                                            const uint64_t* __restrict__ part,
                                                            OutT* __restrict__ out) {
  __shared__ uint64_t sh[kScanThreads / 32 + 1];
  int64_t base = (int64_t)blockIdx.x * kScanChunk + (int64_t)threadIdx.x * kScanPer;
  uint32_t v[kScanPer];
  uint64_t s = 0;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    v[i] = (base + i < n) ? in[base + i] : 0u;
    s += v[i];
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = s;
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t t = 0;
    for (int w = 0; w < kScanThreads / 32; ++w) { uint64_t c = sh[w]; sh[w] = t; t += c; }
  }
  __syncthreads();
  uint64_t run = part[blockIdx.x] + sh[warp] + x - s;
#pragma unroll
  for (int i = 0; i < kScanPer; ++i) {
    if (base + i < n) out[base + i] = (OutT)run;
    run += v[i];
    if (base + i == n - 1) out[n] = (OutT)run;  // total at out[n]
  }
}

template <typename OutT>
static void scan_excl(const uint32_t* in, int64_t n, OutT* out, uint64_t* part, cudaStream_t s) {
  if (n == 0) {
    cudaMemsetAsync(out, 0, sizeof(OutT), s);
    return;
  }
  int64_t nb = ceil_div(n, kScanChunk);
  k_scan_partials<<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, part);
  k_scan_top<<<1, 1024, 0, s>>>(part, nb);
  k_scan_down<OutT><<<(unsigned)nb, kScanThreads, 0, s>>>(in, n, part, out);
  note_launch(3);
}

// ------------------------------------------------------------------ B3: activeCols + patterns + sizes
// One CTA per panel. Pattern bit for entry (row lr of the panel, compacted column q):
// block q / TK, brick (bc = (q % TK) / 4, br = lr / 16), bit = (lr % 16) * 4 + q % 4 (R3).
// Bricks of a block are indexed in CSC order: i = bc * (TM/16) + br.
__global__ void __launch_bounds__(kFillThreads) k_fill(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                      int64_t M, int64_t K, int64_t nnz, int tm, int tk,
                                                      const uint32_t* __restrict__ q,
                                                      const uint32_t* __restrict__ nact_in,
                                                      const uint32_t* __restrict__ brp, uint32_t* __restrict__ ac,
                                                      uint64_t* __restrict__ gpat, uint32_t* __restrict__ blksz) {
  __shared__ int64_t s_rp[129];
  __shared__ unsigned long long s_pat[kFillSmemBricks];
  const int64_t p = blockIdx.x;
  const uint32_t nact = nact_in[p];
  const uint32_t nblk = (nact + tk - 1) / tk;
  if (nblk == 0) return;
  const int64_t b0 = brp[p];
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const int64_t nbricks = (int64_t)nblk * nbk;
  const bool in_smem = nbricks <= kFillSmemBricks;
  unsigned long long* pat = in_smem ? s_pat : reinterpret_cast<unsigned long long*>(gpat + b0 * nbk);
  load_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);
  const int nrows = (int)min((int64_t)tm, M - p * tm);
  for (int64_t i = threadIdx.x; i < nbricks; i += blockDim.x) pat[i] = 0ull;
  __threadfence_block();
  __syncthreads();
  for (int r = 0; r < nrows; ++r) {
    for (int64_t e = s_rp[r] + threadIdx.x; e < s_rp[r + 1]; e += blockDim.x) {
      uint32_t qq = q[e];
      if (qq >= nact) continue;  // only for invalid CSR input
      uint32_t j = qq / tk, lc = qq % tk;
      int bc = lc >> 2, br = r >> 4;
      int bit = ((r & 15) << 2) | (lc & 3);
      atomicOr(&pat[(int64_t)j * nbk + bc * nbrow + br], 1ull << bit);
      ac[(b0 + j) * tk + lc] = (uint32_t)ci[e];
    }
  }
  for (int64_t t = nact + threadIdx.x; t < (int64_t)nblk * tk; t += blockDim.x) ac[b0 * tk + t] = (uint32_t)K;
  __threadfence_block();
  __syncthreads();
  for (int64_t j = threadIdx.x; j < nblk; j += blockDim.x) {
    uint32_t nbr = 0, nz = 0;
    for (int i = 0; i < nbk; ++i) {
      unsigned long long v = in_smem ? pat[j * nbk + i] : __ldcg(&pat[j * nbk + i]);
      nbr += v != 0ull;
      nz += __popcll(v);
      if (in_smem) gpat[(b0 + j) * nbk + i] = v;
    }
    blksz[b0 + j] = block_bytes(nbc, nbr, nz);
  }
}

// ------------------------------------------------------------------ B5: pack HRPB-v1 blocks
__global__ void __launch_bounds__(kFillThreads) k_pack(const int64_t* __restrict__ rp, const float* __restrict__ vals,
                                                      int64_t M, int64_t nnz, int tm, int tk,
                                                      const uint32_t* __restrict__ q,
                                                      const uint32_t* __restrict__ nact_in,
                                                      const uint32_t* __restrict__ brp,
                                                      const uint64_t* __restrict__ gpat,
                                                      const uint64_t* __restrict__ sp, uint8_t* __restrict__ packed) {
  __shared__ int64_t s_rp[129];
  const int64_t p = blockIdx.x;
  const uint32_t nact = nact_in[p];
  const uint32_t nblk = (nact + tk - 1) / tk;
  if (nblk == 0) return;
  const int64_t b0 = brp[p];
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  load_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);
  const int nrows = (int)min((int64_t)tm, M - p * tm);
  // headers, patterns and padding: one thread per block
  for (int64_t j = threadIdx.x; j < nblk; j += blockDim.x) {
    const uint64_t* pt = gpat + (b0 + j) * nbk;
    uint8_t* blk = packed + sp[b0 + j];
    uint32_t nbr = 0, nz = 0;
    for (int i = 0; i < nbk; ++i) { nbr += pt[i] != 0; nz += __popcll(pt[i]); }
    const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
    uint32_t k = 0;
    blk[0] = 0;
    for (int bc = 0; bc < nbc; ++bc) {
      for (int br = 0; br < nbrow; ++br) {
        uint64_t v = pt[bc * nbrow + br];
        if (!v) continue;
        blk[nbc + 1 + k] = (uint8_t)br;                                   // rows[]
        reinterpret_cast<uint64_t*>(blk + hdr)[k] = v;                    // patterns[]
        ++k;
      }
      blk[bc + 1] = (uint8_t)k;                                           // colPtr[]
    }
    for (uint32_t i = nbc + 1 + nbr; i < hdr; ++i) blk[i] = 0;
    const uint32_t end = hdr + 8 * nbr + 4 * nz, size = block_bytes(nbc, nbr, nz);
    for (uint32_t i = end; i < size; ++i) blk[i] = 0;
  }
  // values: destination = values base + prefix popcount of earlier bricks + rank of the bit
  for (int r = 0; r < nrows; ++r) {
    for (int64_t e = s_rp[r] + threadIdx.x; e < s_rp[r + 1]; e += blockDim.x) {
      uint32_t qq = q[e];
      if (qq >= nact) continue;
      uint32_t j = qq / tk, lc = qq % tk;
      int bc = lc >> 2, br = r >> 4;
      int bit = ((r & 15) << 2) | (lc & 3);
      const uint64_t* pt = gpat + (b0 + j) * nbk;
      const int mine = bc * nbrow + br;
      uint32_t nbr = 0, off = 0;
      for (int i = 0; i < nbk; ++i) {
        uint64_t v = pt[i];
        nbr += v != 0;
        if (i < mine) off += __popcll(v);
      }
      const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
      off += __popcll(pt[mine] & ((1ull << bit) - 1ull));
      float* dst = reinterpret_cast<float*>(packed + sp[b0 + j] + hdr + 8 * nbr) + off;
      *dst = vals[e];
    }
  }
}

__global__ void k_finalize(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int64_t P,
                           const uint32_t* __restrict__ brp, const uint64_t* __restrict__ sp,
                           const uint32_t* __restrict__ status, uint64_t* __restrict__ info) {
  uint32_t st = *status;
  if (rp[0] != 0) st |= ST_RP0;
  if (rp[M] != nnz) st |= ST_NNZ;
  uint64_t nb = brp[P];
  info[0] = nb;
  info[1] = sp[nb];
  info[2] = st;
}

// ------------------------------------------------------------------ host orchestration
hrpb_status_t build_impl(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                         const float* values, int32_t tm, int32_t tk, cudaStream_t s, hrpb_handle* h) {
  const int64_t P = ceil_div(M, tm);
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  // upper bounds (no host round trip): sum_p ceil(nact_p/tk) <= nnz/tk + min(P, nnz)
  const int64_t nb_cap = nnz / tk + (P < nnz ? P : nnz);
  const int64_t hdr_cap = align_up(nbc + 1 + nbk, 8) + 15;
  const int64_t brick_cap = nnz < nb_cap * nbk ? nnz : nb_cap * nbk;
  const int64_t bytes_cap = nb_cap * hdr_cap + 8 * brick_cap + 4 * nnz;

  h->M = M; h->K = K; h->nnz = nnz; h->P = P; h->tm = tm; h->tk = tk; h->stream = s;
  h->brp = (uint32_t*)dalloc((P + 1) * sizeof(uint32_t), s);
  h->ac = (uint32_t*)dalloc((nb_cap * tk + 1) * sizeof(uint32_t), s);
  h->sp = (uint64_t*)dalloc((nb_cap + 1) * sizeof(uint64_t), s);
  h->packed = (uint8_t*)dalloc(bytes_cap + 16, s);
  uint32_t* q = (uint32_t*)dalloc((nnz + 1) * sizeof(uint32_t), s);
  uint32_t* nact = (uint32_t*)dalloc((P + 1) * sizeof(uint32_t), s);
  uint32_t* nblk = (uint32_t*)dalloc((P + 1) * sizeof(uint32_t), s);
  uint32_t* blksz = (uint32_t*)dalloc((nb_cap + 1) * sizeof(uint32_t), s);
  uint64_t* gpat = (uint64_t*)dalloc((nb_cap * nbk + 1) * sizeof(uint64_t), s);
  const int64_t nparts = ceil_div((nb_cap > P ? nb_cap : P) + 1, kScanChunk) + 1;
  uint64_t* part = (uint64_t*)dalloc(nparts * sizeof(uint64_t), s);
  uint64_t* info = (uint64_t*)dalloc(4 * sizeof(uint64_t), s);  // [3] = status word
  const int big_ctas = num_sms();
  const int64_t words = ceil_div(K, 32) + 2;
  uint32_t* bigscr = (uint32_t*)dalloc((size_t)big_ctas * 2 * words * sizeof(uint32_t), s);
  hrpb_status_t st = HRPB_SUCCESS;
  if (!h->brp || !h->ac || !h->sp || !h->packed || !q || !nact || !nblk || !blksz || !gpat || !part || !info ||
      !bigscr) {
    st = HRPB_ERROR_OUT_OF_MEMORY;
  }
  uint64_t hinfo[3] = {0, 0, 0};
  if (st == HRPB_SUCCESS) {
    uint32_t* status = reinterpret_cast<uint32_t*>(info + 3);
    cudaMemsetAsync(status, 0, sizeof(uint32_t), s);
    cudaMemsetAsync(blksz, 0, (nb_cap + 1) * sizeof(uint32_t), s);  // tail of the sizePtr scan input
    if (P > 0) {  // B1
      k_rank_small<<<(unsigned)P, kSmallThreads, 0, s>>>(row_ptr, col_idx, M, K, nnz, tm, tk, q, nact, nblk, status);
      k_rank_big<<<big_ctas, kBigThreads, 0, s>>>(row_ptr, col_idx, M, K, nnz, tm, tk, P, q, nact, nblk, bigscr,
                                                   words, status);
      note_launch(2);
    }
    scan_excl<uint32_t>(nblk, P, h->brp, part, s);  // B2: blockedRowPtr
    if (P > 0) {                                     // B3
      k_fill<<<(unsigned)P, kFillThreads, 0, s>>>(row_ptr, col_idx, M, K, nnz, tm, tk, q, nact, h->brp, h->ac, gpat,
                                                  blksz);
      note_launch();
    }
    scan_excl<uint64_t>(blksz, nb_cap, h->sp, part, s);  // B4: sizePtr (entries past NUM_BLKS are zero)
    if (P > 0) {                                          // B5
      k_pack<<<(unsigned)P, kFillThreads, 0, s>>>(row_ptr, values, M, nnz, tm, tk, q, nact, h->brp, gpat, h->sp,
                                                  h->packed);
      note_launch();
    }
    k_finalize<<<1, 1, 0, s>>>(row_ptr, M, nnz, P, h->brp, h->sp, status, info);
    note_launch();
    cudaError_t e = cudaMemcpyAsync(hinfo, info, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_status(e);
  }
  dfree(q, s); dfree(nact, s); dfree(nblk, s); dfree(blksz, s); dfree(gpat, s); dfree(part, s); dfree(info, s);
  dfree(bigscr, s);
  if (st == HRPB_SUCCESS && hinfo[2] != 0) st = HRPB_ERROR_INVALID_CSR;
  h->NB = (int64_t)hinfo[0];
  h->bytes = (int64_t)hinfo[1];
  return st;
}

}  // namespace hrpb
