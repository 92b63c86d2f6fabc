// build.cu — GPU CSR -> HRPB builder, bit-identical to the oracle.
//
// Paper: Alg. "CSR to HRPB Phase1/Phase2" runs on the host with OpenMP over panel
// chunks and prefix sums; §"HRPB Sparse Matrix Data structure" defines the output.
// B200 design: no host round trip until the end; outputs are allocated at
// upper bounds computable from (M, nnz), so the pipeline is
//   k_count / k_count_big  (B1 + B3 counting: per-panel sorted-unique active columns -> compacted
//                           rank q of every entry, nact; brick patterns; block sizes; CSR validation)
//   scan(nblk) -> blockedRowPtr (B2); scan(panel bytes) -> panel byte offsets (B4, panel level)
//   k_emit                 (B3 + B4 + B5: activeCols with sentinel K, sizePtr, HRPB-v1 headers,
//                           patterns, values in brick-CSC / row-major order)
//   k_finalize             (NUM_BLKS, byte total, status) -> one 32-byte D2H read + sync.
// Panel p keeps its brick patterns between the two passes in a scratch region addressed from its
// first entry offset, base(p) = floor(e0 * nbk / tk) + 2 p nbk, which never overlaps the next panel's.
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
constexpr int kSmallCap = 2048;      // entries per panel handled in shared memory
constexpr int kSpanWords = 512;      // bitmap ranking when the panel's column span <= 16384
constexpr int kBigThreads = 512;
constexpr int kEmitThreads = 128;
constexpr int kWarpCap = 256;        // entries per panel handled by one warp (no CTA barriers)
constexpr int kWarpSpanWords = 256;  // warp bitmap ranking when the column span < 8192 (bitmap + prefix = s_keys)
constexpr int kWarpsPerCta = 8;
constexpr int kWarpCap2 = 1024;      // second warp pass (listed panels, bitmap ranking only)

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

// ------------------------------------------------------------------ pass A, warp per panel
// One warp per panel, no CTA barriers: entries live in registers (CAP/32 per lane), ranks come from a
// per-warp bitmap (column span < 8192) or, when SORT, a warp bitonic sort; patterns via 32-bit shared
// atomics. Returns 0 when the panel was counted, 1 when it has more than CAP entries, 2 when its column
// span needs the sort path and SORT is off.
template <int CAP, bool SORT>
__device__ __forceinline__ int count_panel_warp(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                int64_t M, int64_t K, int64_t nnz, int tm, int tk, int64_t p,
                                                uint32_t* __restrict__ q, uint32_t* __restrict__ nact_out,
                                                uint32_t* __restrict__ nblk_out, uint32_t* __restrict__ pbytes_out,
                                                uint64_t* __restrict__ gpat, uint32_t* status, uint8_t* my,
                                                int64_t& E_out) {
  constexpr int PER = CAP / 32;
  const int lane = threadIdx.x & 31;
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(my);                           // SORT ? [CAP] : bitmap 2 KB
  constexpr int kKeyBytes = SORT ? CAP * 8 : 2 * kWarpSpanWords * 4;
  uint32_t* s_qb = reinterpret_cast<uint32_t*>(my + kKeyBytes);                  // SORT ? [CAP] : none
  int64_t* s_rp = reinterpret_cast<int64_t*>(my + kKeyBytes + (SORT ? CAP * 4 : 0));  // [tm + 1]
  unsigned long long* s_pat = reinterpret_cast<unsigned long long*>(s_rp + ((tm + 2) & ~1));
  warp_panel_rows(rp, M, nnz, tm, p, s_rp, status);
  const int nrows = (int)min((int64_t)tm, M - p * tm);
  const int64_t e0 = s_rp[0];
  const int64_t E64 = s_rp[nrows] - e0;
  E_out = E64;
  if (E64 > CAP) return 1;
  static_assert(2 * kWarpSpanWords * 4 <= kKeyBytes, "bitmap + prefix must fit in s_keys");
  const int E = (int)E64;
  if (E == 0) {
    if (lane == 0) { nact_out[p] = 0; nblk_out[p] = 0; pbytes_out[p] = 0; }
    return 0;
  }
  uint32_t col[PER];
  int rowv[PER];
  int32_t mn = INT32_MAX, mx = INT32_MIN;
  bool bad_range = false, bad_order = false;
#pragma unroll
  for (int k = 0; k < PER; ++k) {  // all loads first
    const int idx = lane + 32 * k;
    col[k] = idx < E ? (uint32_t)ci[e0 + idx] : 0u;
  }
  uint32_t prev_last = 0;  // column of entry 32k - 1 (lane 31 of the previous k)
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const int idx = lane + 32 * k;
    uint32_t prevc = __shfl_up_sync(0xffffffffu, col[k], 1);
    if (lane == 0) prevc = prev_last;
    prev_last = __shfl_sync(0xffffffffu, col[k], 31);
    rowv[k] = 0;
    if (idx < E) {
      const int64_t e = e0 + idx;
      const int32_t c = (int32_t)col[k];
      const int r = row_of(s_rp, nrows, e);
      rowv[k] = r;
      bad_range |= c < 0 || c >= K;
      if (e > s_rp[r] && (int32_t)prevc >= c) bad_order = true;
      mn = min(mn, c);
      mx = max(mx, c);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  const bool small_span = (int64_t)mx - (int64_t)mn < 32 * kWarpSpanWords;
  if (!SORT && !small_span) return 2;  // (warp-uniform) handled by the CTA path
  if (__any_sync(0xffffffffu, bad_range) && lane == 0) atomicOr(status, ST_COL_RANGE);
  if (__any_sync(0xffffffffu, bad_order) && lane == 0) atomicOr(status, ST_COL_ORDER);
  uint32_t qv[PER];
  uint32_t nact = 0;
  if (small_span) {
    uint32_t* bm = reinterpret_cast<uint32_t*>(s_keys);
    uint32_t* pre = bm + kWarpSpanWords;
    constexpr int kW = kWarpSpanWords / 32;
#pragma unroll
    for (int i = 0; i < kW; ++i) bm[lane * kW + i] = 0;
    __syncwarp();
#pragma unroll
    for (int k = 0; k < PER; ++k)
      if (lane + 32 * k < E) {
        const uint32_t off = col[k] - (uint32_t)mn;
        atomicOr(&bm[off >> 5], 1u << (off & 31));
      }
    __syncwarp();
    uint32_t cnt[kW], sum = 0;
#pragma unroll
    for (int i = 0; i < kW; ++i) { cnt[i] = __popc(bm[lane * kW + i]); sum += cnt[i]; }
    uint32_t run = warp_excl_scan(sum, &nact);
#pragma unroll
    for (int i = 0; i < kW; ++i) { pre[lane * kW + i] = run; run += cnt[i]; }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const uint32_t off = col[k] - (uint32_t)mn;
      const uint32_t w = (off >> 5) & (kWarpSpanWords - 1), b = off & 31;
      qv[k] = pre[w] + __popc(bm[w] & ((1u << b) - 1u));
    }
  } else if constexpr (SORT) {
    int n = 32;
    while (n < E) n <<= 1;
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int idx = lane + 32 * k;
      if (idx < n) s_keys[idx] = idx < E ? ((uint64_t)col[k] << 32) | (uint32_t)idx : ~0ull;
    }
    __syncwarp();
    for (int kk = 2; kk <= n; kk <<= 1) {
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < n; i += 32) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const uint64_t a = s_keys[i], b = s_keys[ixj];
            if ((a > b) == ((i & kk) == 0)) { s_keys[i] = b; s_keys[ixj] = a; }
          }
        }
        __syncwarp();
      }
    }
    const int per = n / 32;
    const int beg = lane * per;
    uint32_t sum = 0;
    for (int i = beg; i < beg + per && i < E; ++i)
      if (i == 0 || (s_keys[i] >> 32) != (s_keys[i - 1] >> 32)) ++sum;
    uint32_t run = warp_excl_scan(sum, &nact);
    for (int i = beg; i < beg + per && i < E; ++i) {
      if (i == 0 || (s_keys[i] >> 32) != (s_keys[i - 1] >> 32)) ++run;
      s_qb[(uint32_t)s_keys[i]] = run - 1;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < PER; ++k) qv[k] = lane + 32 * k < E ? s_qb[lane + 32 * k] : 0u;
  }
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const uint32_t nblk = (nact + tk - 1) / tk;
  const int nbricks = (int)nblk * nbk;
  for (int i = lane; i < nbricks; i += 32) s_pat[i] = 0ull;
  __syncwarp();
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    if (lane + 32 * k < E) {
      const uint32_t qq = qv[k], r = (uint32_t)rowv[k];
      const uint32_t j = qq / tk, lc = qq % tk;
      const int bit = (int)(((r & 15) << 2) | (lc & 3));
      uint32_t* half = reinterpret_cast<uint32_t*>(&s_pat[j * nbk + (lc >> 2) * nbrow + (r >> 4)]) + (bit >> 5);
      atomicOr(half, 1u << (bit & 31));
      q[e0 + lane + 32 * k] = qq;
    }
  }
  __syncwarp();
  uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
  for (int i = lane; i < nbricks; i += 32) gp[i] = s_pat[i];
  uint32_t bytes = 0;
  for (uint32_t j = lane; j < nblk; j += 32) {
    uint32_t nbr = 0, nz = 0;
    for (int i = 0; i < nbk; ++i) { const uint64_t v = s_pat[j * nbk + i]; nbr += v != 0ull; nz += __popcll(v); }
    bytes += block_bytes(nbc, nbr, nz);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bytes += __shfl_xor_sync(0xffffffffu, bytes, o);
  if (lane == 0) { nact_out[p] = nact; nblk_out[p] = nblk; pbytes_out[p] = bytes; }
  return 0;
}

template <int CAP, bool SORT>
__host__ __device__ constexpr int count_warp_smem(int tm, int tk) {
  return (int)((((SORT ? CAP * 12 : 2 * kWarpSpanWords * 4) + ((tm + 2) & ~1) * 8 + (CAP / tk) * (tk / 4) * (tm / 16) * 8) +
                15) & ~15);
}

// Warp per panel over all panels (CAP = 256, sort allowed); panels with more entries go to list L1.
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_count_warp(
    const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t M, int64_t K, int64_t nnz, int tm,
    int tk, int64_t P, uint32_t* __restrict__ q, uint32_t* __restrict__ nact_out, uint32_t* __restrict__ nblk_out,
    uint32_t* __restrict__ pbytes_out, uint64_t* __restrict__ gpat, uint32_t* __restrict__ l1, uint32_t* __restrict__ nl1,
    uint32_t* status) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int wid = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * kWarpsPerCta + wid;
  if (p >= P) return;
  uint8_t* my = dsm + (size_t)wid * count_warp_smem<kWarpCap, true>(tm, tk);
  int64_t E;
  const int r = count_panel_warp<kWarpCap, true>(rp, ci, M, K, nnz, tm, tk, p, q, nact_out, nblk_out, pbytes_out,
                                                  gpat, status, my, E);
  if (r != 0 && (threadIdx.x & 31) == 0) l1[atomicAdd(nl1, 1u)] = (uint32_t)p;
}

// Warp per listed panel (CAP = 1024, bitmap ranking only). Not handled -> list L2 (CTA count); more than
// kWarpCap2 entries -> also list L3 (CTA emit).
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_count_warp2(
    const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, int64_t M, int64_t K, int64_t nnz, int tm,
    int tk, uint32_t* __restrict__ q, uint32_t* __restrict__ nact_out, uint32_t* __restrict__ nblk_out,
    uint32_t* __restrict__ pbytes_out, uint64_t* __restrict__ gpat, const uint32_t* __restrict__ l1,
    const uint32_t* __restrict__ nl1, uint32_t* __restrict__ l2, uint32_t* __restrict__ nl2,
    uint32_t* __restrict__ l3, uint32_t* __restrict__ nl3, uint32_t* status) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint8_t* my = dsm + (size_t)wid * count_warp_smem<kWarpCap2, false>(tm, tk);
  const uint32_t count = *nl1;
  for (uint32_t t = blockIdx.x * kWarpsPerCta + wid; t < count; t += gridDim.x * kWarpsPerCta) {
    const int64_t p = l1[t];
    int64_t E;
    const int r = count_panel_warp<kWarpCap2, false>(rp, ci, M, K, nnz, tm, tk, p, q, nact_out, nblk_out,
                                                      pbytes_out, gpat, status, my, E);
    if (lane == 0) {
      if (r != 0) l2[atomicAdd(nl2, 1u)] = (uint32_t)p;
      if (E > kWarpCap2) l3[atomicAdd(nl3, 1u)] = (uint32_t)p;
    }
    __syncwarp();
  }
}

// ------------------------------------------------------------------ pass B, warp per panel
template <int CAP>
__device__ __forceinline__ void emit_panel_warp(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                const float* __restrict__ vals, int64_t M, int64_t K, int64_t nnz,
                                                int tm, int tk, int64_t p, const uint32_t* __restrict__ q,
                                                const uint32_t* __restrict__ nact_in,
                                                const uint32_t* __restrict__ brp, const uint64_t* __restrict__ poff,
                                                const uint64_t* __restrict__ gpat, uint32_t* __restrict__ ac,
                                                uint64_t* __restrict__ sp, uint8_t* __restrict__ packed, uint8_t* my) {
  const int lane = threadIdx.x & 31;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const uint32_t b0 = brp[p], nblk = brp[p + 1] - b0;
  if (nblk == 0) return;
  int64_t* s_rp = reinterpret_cast<int64_t*>(my);
  uint64_t* s_vbase = reinterpret_cast<uint64_t*>(s_rp + ((tm + 2) & ~1));  // [CAP / 16]
  uint64_t* s_pt = s_vbase + CAP / 16;                                     // [CAP / tk * nbk]
  uint16_t* s_soff = reinterpret_cast<uint16_t*>(s_pt + (CAP / tk) * nbk); // value offset of each brick slot
  warp_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);
  const int nrows = (int)min((int64_t)tm, M - p * tm);
  const uint32_t nact = nact_in[p];
  const int64_t e0 = s_rp[0], e1 = s_rp[nrows];
  const uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
  for (int i = lane; i < (int)nblk * nbk; i += 32) s_pt[i] = gp[i];
  __syncwarp();
  uint64_t carry = poff[p];
  for (uint32_t c0 = 0; c0 < nblk; c0 += 32) {  // blocks, 32 at a time (one per lane)
    const uint32_t j = c0 + lane;
    uint32_t nbr = 0, nz = 0, size = 0;
    if (j < nblk) {
      for (int i = 0; i < nbk; ++i) {
        const uint64_t v = s_pt[j * nbk + i];
        s_soff[j * nbk + i] = (uint16_t)nz;  // popcount of the earlier slots (CSC order)
        nbr += v != 0ull;
        nz += __popcll(v);
      }
      size = block_bytes(nbc, nbr, nz);
    }
    uint32_t tot;
    const uint64_t off = carry + warp_excl_scan(size, &tot);
    if (j < nblk) {
      sp[b0 + j] = off;
      uint8_t* blk = packed + off;
      const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
      uint32_t k = 0;
      blk[0] = 0;
      for (int bc = 0; bc < nbc; ++bc) {
        for (int br = 0; br < nbrow; ++br) {
          const uint64_t v = s_pt[j * nbk + bc * nbrow + br];
          if (!v) continue;
          blk[nbc + 1 + k] = (uint8_t)br;
          reinterpret_cast<uint64_t*>(blk + hdr)[k] = v;
          ++k;
        }
        blk[bc + 1] = (uint8_t)k;
      }
      for (uint32_t i = nbc + 1 + nbr; i < hdr; ++i) blk[i] = 0;
      for (uint32_t i = hdr + 8 * nbr + 4 * nz; i < size; ++i) blk[i] = 0;
      s_vbase[j] = off + hdr + 8 * nbr;
    }
    carry += tot;
  }
  for (int64_t t = nact + lane; t < (int64_t)nblk * tk; t += 32) ac[(int64_t)b0 * tk + t] = (uint32_t)K;
  __syncwarp();
  constexpr int kBatch = 8;  // loads of 8 rounds in flight before any use
  for (int64_t eb = e0; eb < e1; eb += 32 * kBatch) {
    uint32_t qb[kBatch];
    int32_t cb[kBatch];
    float vb[kBatch];
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int64_t e = eb + 32 * u + lane;
      qb[u] = e < e1 ? q[e] : 0xFFFFFFFFu;
      cb[u] = e < e1 ? ci[e] : 0;
      vb[u] = e < e1 ? vals[e] : 0.f;
    }
#pragma unroll
    for (int u = 0; u < kBatch; ++u) {
      const int64_t e = eb + 32 * u + lane;
      const uint32_t qq = qb[u];
      if (qq >= nact) continue;  // past the panel, or invalid CSR input
      const int r = row_of(s_rp, nrows, e);
      const uint32_t jb = qq / tk, lc = qq % tk;
      ac[((int64_t)b0 + jb) * tk + lc] = (uint32_t)cb[u];
      const int bit = ((r & 15) << 2) | (lc & 3);
      const int mine = (lc >> 2) * nbrow + (r >> 4);
      const uint32_t o = s_soff[jb * nbk + mine] + __popcll(s_pt[jb * nbk + mine] & ((1ull << bit) - 1ull));
      reinterpret_cast<float*>(packed + s_vbase[jb])[o] = vb[u];
    }
  }
  __syncwarp();
}

template <int CAP>
__host__ __device__ constexpr int emit_warp_smem(int tm, int tk) {
  return (int)((((tm + 2) & ~1) * 8 + (CAP / 16) * 8 + (CAP / tk) * (tk / 4) * (tm / 16) * (8 + 2) + 15) & ~15);
}

__device__ __forceinline__ int64_t panel_entries(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int tm,
                                                 int64_t p) {
  const int64_t r0 = p * tm;
  const int nrows = (int)min((int64_t)tm, M - r0);
  int64_t a = rp[r0], b = rp[r0 + nrows];
  a = a < 0 ? 0 : (a > nnz ? nnz : a);
  b = b < 0 ? 0 : (b > nnz ? nnz : b);
  return b - a;
}

// all panels with <= kWarpCap entries
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_emit_warp(
    const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const float* __restrict__ vals, int64_t M,
    int64_t K, int64_t nnz, int tm, int tk, int64_t P, const uint32_t* __restrict__ q,
    const uint32_t* __restrict__ nact_in, const uint32_t* __restrict__ brp, const uint64_t* __restrict__ poff,
    const uint64_t* __restrict__ gpat, uint32_t* __restrict__ ac, uint64_t* __restrict__ sp,
    uint8_t* __restrict__ packed) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int wid = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * kWarpsPerCta + wid;
  if (p >= P) return;
  if (panel_entries(rp, M, nnz, tm, p) > kWarpCap) return;  // listed in L1 (k_emit_warp2 / k_emit)
  emit_panel_warp<kWarpCap>(rp, ci, vals, M, K, nnz, tm, tk, p, q, nact_in, brp, poff, gpat, ac, sp, packed,
                            dsm + (size_t)wid * emit_warp_smem<kWarpCap>(tm, tk));
}

// listed panels (L1) with <= kWarpCap2 entries
__global__ void __launch_bounds__(32 * kWarpsPerCta) k_emit_warp2(
    const int64_t* __restrict__ rp, const int32_t* __restrict__ ci, const float* __restrict__ vals, int64_t M,
    int64_t K, int64_t nnz, int tm, int tk, const uint32_t* __restrict__ q, const uint32_t* __restrict__ nact_in,
    const uint32_t* __restrict__ brp, const uint64_t* __restrict__ poff, const uint64_t* __restrict__ gpat,
    uint32_t* __restrict__ ac, uint64_t* __restrict__ sp, uint8_t* __restrict__ packed,
    const uint32_t* __restrict__ l1, const uint32_t* __restrict__ nl1) {
  extern __shared__ __align__(16) uint8_t dsm[];
  const int wid = threadIdx.x >> 5;
  uint8_t* my = dsm + (size_t)wid * emit_warp_smem<kWarpCap2>(tm, tk);
  const uint32_t count = *nl1;
  for (uint32_t t = blockIdx.x * kWarpsPerCta + wid; t < count; t += gridDim.x * kWarpsPerCta) {
    const int64_t p = l1[t];
    if (panel_entries(rp, M, nnz, tm, p) > kWarpCap2) continue;  // listed in L3 (k_emit)
    emit_panel_warp<kWarpCap2>(rp, ci, vals, M, K, nnz, tm, tk, p, q, nact_in, brp, poff, gpat, ac, sp, packed, my);
  }
}

// ------------------------------------------------------------------ pass A, kWarpCap < entries <= kSmallCap
// One CTA per listed panel ("for row_panel in rowPanels_chunk"). q[e] = rank of col_idx[e] among the
// panel's distinct columns (ascending, R23; "active_cols = uniq(cols[...])"), nblk = ceil(nact/TK)
// (R1), brick patterns (bit = (r % 16) * 4 + q % 4, R3) and the panel's total block bytes.
__global__ void __launch_bounds__(kSmallThreads) k_count(const int64_t* __restrict__ rp,
                                                        const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                        int64_t nnz, int tm, int tk, uint32_t* __restrict__ q,
                                                        uint32_t* __restrict__ nact_out,
                                                        uint32_t* __restrict__ nblk_out,
                                                        uint32_t* __restrict__ pbytes_out,
                                                        uint64_t* __restrict__ gpat,
                                                        const uint32_t* __restrict__ midlist,
                                                        const uint32_t* __restrict__ nmid,
                                                        uint32_t* __restrict__ biglist,
                                                        uint32_t* __restrict__ nbig, uint32_t* status) {
  extern __shared__ __align__(16) uint8_t dsm[];
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_scan[kSmallThreads / 32 + 1];
  __shared__ int32_t s_mm[2 * kSmallThreads / 32];
  uint64_t* s_keys = reinterpret_cast<uint64_t*>(dsm);                 // [kSmallCap] (also the bitmap)
  uint32_t* s_col = reinterpret_cast<uint32_t*>(s_keys + kSmallCap);   // [kSmallCap]
  uint32_t* s_q = s_col + kSmallCap;                                   // [kSmallCap]
  uint8_t* s_row = reinterpret_cast<uint8_t*>(s_q + kSmallCap);        // [kSmallCap]
  unsigned long long* s_pat = reinterpret_cast<unsigned long long*>(s_row + kSmallCap);  // [cap bricks]

  const uint32_t count = *nmid;
  for (uint32_t t = blockIdx.x; t < count; t += gridDim.x) {
  const int64_t p = midlist[t];
  load_panel_rows(rp, M, nnz, tm, p, s_rp, status);
  const int nrows = (int)min((int64_t)tm, M - p * tm);
  const int64_t e0 = s_rp[0];
  const int E = (int)min((int64_t)kSmallCap + 1, s_rp[nrows] - e0);
  if (E > kSmallCap) {  // CTA-uniform: handled by k_count_big
    if (threadIdx.x == 0) biglist[atomicAdd(nbig, 1u)] = (uint32_t)p;
    continue;
  }
  // entries -> shared memory (local row, column)
  int32_t mn = INT32_MAX, mx = INT32_MIN;
  for (int i = threadIdx.x; i < E; i += blockDim.x) {  // one flat pass: all loads in flight together
    const int32_t c = ci[e0 + i];
    s_col[i] = (uint32_t)c;
    s_row[i] = (uint8_t)row_of(s_rp, nrows, e0 + i);
    mn = min(mn, c);
    mx = max(mx, c);
  }
  block_minmax<kSmallThreads>(mn, mx, s_mm);  // (contains __syncthreads)
  for (int i = threadIdx.x; i < E; i += blockDim.x) {  // validation
    const int32_t c = (int32_t)s_col[i];
    if (c < 0 || c >= K) atomicOr(status, ST_COL_RANGE);
    if (i > 0 && s_row[i - 1] == s_row[i] && (int32_t)s_col[i - 1] >= c) atomicOr(status, ST_COL_ORDER);
  }
  uint32_t nact = 0;
  const int64_t span = (int64_t)mx - (int64_t)mn + 1;
  if (span <= 32 * kSpanWords) {
    // bitmap ranking: set bits, exclusive popcount prefix per word, rank = prefix + popc(word & below)
    uint32_t* bm = reinterpret_cast<uint32_t*>(s_keys);
    uint32_t* pre = bm + kSpanWords;
    for (int i = threadIdx.x; i < kSpanWords; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
      const uint32_t off = s_col[i] - (uint32_t)mn;
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
    for (int i = threadIdx.x; i < E; i += blockDim.x) {
      const uint32_t off = s_col[i] - (uint32_t)mn;
      const uint32_t w = off >> 5, b = off & 31;
      s_q[i] = pre[w] + __popc(bm[w] & ((1u << b) - 1u));
    }
  } else {
    // sort ranking: bitonic sort of (col << 32 | local index), unique flags, scan
    int n = 32;
    while (n < E) n <<= 1;
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      s_keys[i] = i < E ? ((uint64_t)s_col[i] << 32) | (uint32_t)i : ~0ull;
    __syncthreads();
    for (int k = 2; k <= n; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const uint64_t a = s_keys[i], b = s_keys[ixj];
            if ((a > b) == ((i & k) == 0)) { s_keys[i] = b; s_keys[ixj] = a; }
          }
        }
        __syncthreads();
      }
    }
    const int per = n / kSmallThreads > 0 ? n / kSmallThreads : 1;
    const int beg = threadIdx.x * per;
    uint32_t sum = 0;
    for (int i = beg; i < beg + per && i < E; ++i)
      if (i == 0 || (s_keys[i] >> 32) != (s_keys[i - 1] >> 32)) ++sum;
    uint32_t run = block_excl_scan<kSmallThreads>(sum, &nact, s_scan);
    for (int i = beg; i < beg + per && i < E; ++i) {
      if (i == 0 || (s_keys[i] >> 32) != (s_keys[i - 1] >> 32)) ++run;
      s_q[(uint32_t)s_keys[i]] = run - 1;
    }
  }
  // patterns (fill_brick_nnz_pattern): brick i = bc * (TM/16) + br in CSC order
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const uint32_t nblk = (nact + tk - 1) / tk;
  const int nbricks = (int)nblk * nbk;
  for (int i = threadIdx.x; i < nbricks; i += blockDim.x) s_pat[i] = 0ull;
  __syncthreads();
  for (int i = threadIdx.x; i < E; i += blockDim.x) {
    const uint32_t qq = s_q[i], r = s_row[i];
    const uint32_t j = qq / tk, lc = qq % tk;
    const int bit = (int)(((r & 15) << 2) | (lc & 3));
    // 32-bit OR on the half holding the bit (a 64-bit shared atomicOr is a CAS loop on sm_100)
    uint32_t* half = reinterpret_cast<uint32_t*>(&s_pat[j * nbk + (lc >> 2) * nbrow + (r >> 4)]) + (bit >> 5);
    atomicOr(half, 1u << (bit & 31));
    q[e0 + i] = qq;
  }
  __syncthreads();
  uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
  for (int i = threadIdx.x; i < nbricks; i += blockDim.x) gp[i] = s_pat[i];
  uint32_t bytes = 0;
  for (uint32_t j = threadIdx.x; j < nblk; j += blockDim.x) {
    uint32_t nbr = 0, nz = 0;
    for (int i = 0; i < nbk; ++i) { const uint64_t v = s_pat[j * nbk + i]; nbr += v != 0ull; nz += __popcll(v); }
    bytes += block_bytes(nbc, nbr, nz);
  }
  uint32_t total;
  block_excl_scan<kSmallThreads>(bytes, &total, s_scan);
  if (threadIdx.x == 0) { nact_out[p] = nact; nblk_out[p] = nblk; pbytes_out[p] = total; }
  }  // panel loop
}

// ------------------------------------------------------------------ pass A, panels with > kSmallCap entries
// Persistent CTAs over the hub-panel list; each CTA owns a global bitmap over the panel's column span.
__global__ void __launch_bounds__(kBigThreads) k_count_big(const int64_t* __restrict__ rp,
                                                          const int32_t* __restrict__ ci, int64_t M, int64_t K,
                                                          int64_t nnz, int tm, int tk, uint32_t* __restrict__ q,
                                                          uint32_t* __restrict__ nact_out,
                                                          uint32_t* __restrict__ nblk_out,
                                                          uint32_t* __restrict__ pbytes_out,
                                                          uint64_t* __restrict__ gpat,
                                                          const uint32_t* __restrict__ biglist,
                                                          const uint32_t* __restrict__ nbig, uint32_t* scratch,
                                                          int64_t words_per_cta, uint32_t* status) {
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_scan[kBigThreads / 32 + 1];
  __shared__ int32_t s_mm[2 * kBigThreads / 32];
  uint32_t* bm = scratch + (int64_t)blockIdx.x * 2 * words_per_cta;
  uint32_t* pre = bm + words_per_cta;
  const uint32_t count = *nbig;
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  for (uint32_t t = blockIdx.x; t < count; t += gridDim.x) {
    const int64_t p = biglist[t];
    load_panel_rows(rp, M, nnz, tm, p, s_rp, status);
    const int nrows = (int)min((int64_t)tm, M - p * tm);
    const int64_t e0 = s_rp[0], e1 = s_rp[nrows];
    int32_t mn = INT32_MAX, mx = INT32_MIN;
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int32_t c = ci[e];
      const bool ok = c >= 0 && c < K;
      if (!ok) atomicOr(status, ST_COL_RANGE);
      const int r = row_of(s_rp, nrows, e);
      if (e > s_rp[r] && ci[e - 1] >= c) atomicOr(status, ST_COL_ORDER);
      if (ok) { mn = min(mn, c); mx = max(mx, c); }
    }
    block_minmax<kBigThreads>(mn, mx, s_mm);
    if (mn > mx) { mn = 0; mx = 0; }
    const int64_t base = mn >> 5;
    const int64_t W = (mx >> 5) - base + 1;
    for (int64_t i = threadIdx.x; i < W; i += blockDim.x) bm[i] = 0;
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int32_t c = ci[e];
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
    const uint32_t nblk = (nact + tk - 1) / tk;
    unsigned long long* gp = reinterpret_cast<unsigned long long*>(gpat + pat_base(e0, p, nbk, tk));
    for (int64_t i = threadIdx.x; i < (int64_t)nblk * nbk; i += blockDim.x) gp[i] = 0ull;
    __threadfence_block();
    __syncthreads();
    for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const int32_t c = ci[e];
      if (c < 0 || c >= K) { q[e] = 0xFFFFFFFFu; continue; }
      const int r = row_of(s_rp, nrows, e);
      const int64_t w = (c >> 5) - base;
      const uint32_t qq = __ldcg(&pre[w]) + __popc(__ldcg(&bm[w]) & ((1u << (c & 31)) - 1u));
      q[e] = qq;
      const uint32_t j = qq / tk, lc = qq % tk;
      atomicOr(&gp[(int64_t)j * nbk + (lc >> 2) * nbrow + (r >> 4)], 1ull << (((r & 15) << 2) | (lc & 3)));
    }
    __threadfence_block();
    __syncthreads();
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
    uint32_t total;
    block_excl_scan<kBigThreads>(bytes, &total, s_scan);
    if (threadIdx.x == 0) { nact_out[p] = nact; nblk_out[p] = nblk; pbytes_out[p] = total; }
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

// ------------------------------------------------------------------ pass B (CTA), panels with > kWarpCap entries
// One CTA per listed panel. Block j of panel p is global block b0 + j (b0 = blockedRowPtr[p]); its byte offset
// is the panel offset plus the in-panel exclusive scan of block sizes (sizePtr). Header,
// patterns and values follow the HRPB-v1 layout; value destination = values base + popcount of the
// earlier bricks + popcount of the lower bits of its own brick.
__global__ void __launch_bounds__(kEmitThreads) k_emit(const int64_t* __restrict__ rp, const int32_t* __restrict__ ci,
                                                      const float* __restrict__ vals, int64_t M, int64_t K,
                                                      int64_t nnz, int tm, int tk, const uint32_t* __restrict__ q,
                                                      const uint32_t* __restrict__ nact_in,
                                                      const uint32_t* __restrict__ brp,
                                                      const uint64_t* __restrict__ poff,
                                                      const uint64_t* __restrict__ gpat, uint32_t* __restrict__ ac,
                                                      uint64_t* __restrict__ sp, uint8_t* __restrict__ packed,
                                                      const uint32_t* __restrict__ midlist,
                                                      const uint32_t* __restrict__ nmid) {
  __shared__ int64_t s_rp[129];
  __shared__ uint32_t s_scan[kEmitThreads / 32 + 1];
  __shared__ uint64_t s_vbase[kEmitThreads];     // byte offset of each block's values (single-chunk panels)
  __shared__ uint64_t s_pt[kEmitThreads * 4];    // patterns (single-chunk panels with nbk <= 4)
  const uint32_t count = *nmid;
  for (uint32_t tt = blockIdx.x; tt < count; tt += gridDim.x) {
  const int64_t p = midlist[tt];
  const uint32_t b0 = brp[p], nblk = brp[p + 1] - b0;
  if (nblk == 0) continue;
  const uint32_t nact = nact_in[p];
  load_panel_rows(rp, M, nnz, tm, p, s_rp, nullptr);
  const int nrows = (int)min((int64_t)tm, M - p * tm);
  const int64_t e0 = s_rp[0];
  const int nbc = tk / HRPB_BRICK_K, nbrow = tm / HRPB_BRICK_M, nbk = nbc * nbrow;
  const uint64_t* gp = gpat + pat_base(e0, p, nbk, tk);
  // blocks: sizes, sizePtr, headers, patterns, padding (chunks of kEmitThreads blocks)
  uint64_t carry = poff[p];
  for (uint32_t c0 = 0; c0 < nblk; c0 += kEmitThreads) {
    const uint32_t j = c0 + threadIdx.x;
    uint32_t nbr = 0, nz = 0, size = 0;
    if (j < nblk) {
      for (int i = 0; i < nbk; ++i) {
        const uint64_t v = gp[(int64_t)j * nbk + i];
        nbr += v != 0ull;
        nz += __popcll(v);
      }
      size = block_bytes(nbc, nbr, nz);
    }
    uint32_t tot;
    const uint32_t ex = block_excl_scan<kEmitThreads>(size, &tot, s_scan);
    if (j < nblk) {
      const uint64_t off = carry + ex;
      sp[b0 + j] = off;
      uint8_t* blk = packed + off;
      const uint64_t* pt = gp + (int64_t)j * nbk;
      const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
      uint32_t k = 0;
      blk[0] = 0;
      for (int bc = 0; bc < nbc; ++bc) {
        for (int br = 0; br < nbrow; ++br) {
          const uint64_t v = pt[bc * nbrow + br];
          if (!v) continue;
          blk[nbc + 1 + k] = (uint8_t)br;                 // rows[]
          reinterpret_cast<uint64_t*>(blk + hdr)[k] = v;  // patterns[]
          ++k;
        }
        blk[bc + 1] = (uint8_t)k;  // colPtr[]
      }
      for (uint32_t i = nbc + 1 + nbr; i < hdr; ++i) blk[i] = 0;
      for (uint32_t i = hdr + 8 * nbr + 4 * nz; i < size; ++i) blk[i] = 0;
      if (nblk <= kEmitThreads) {
        s_vbase[j] = off + hdr + 8 * nbr;
        if (nbk <= 4)
          for (int i = 0; i < nbk; ++i) s_pt[j * nbk + i] = pt[i];
      }
    }
    carry += tot;
  }
  for (int64_t t = nact + threadIdx.x; t < (int64_t)nblk * tk; t += blockDim.x) ac[(int64_t)b0 * tk + t] = (uint32_t)K;
  __syncthreads();  // sizePtr entries / staged metadata of this panel are visible to the whole CTA
  const bool staged = nblk <= kEmitThreads && nbk <= 4;
  const int64_t e1 = s_rp[nrows];
  for (int64_t e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    const uint32_t qq = q[e];
    const int32_t c = ci[e];
    const float v = vals[e];
    if (qq >= nact) continue;  // only for invalid CSR input
    const int r = row_of(s_rp, nrows, e);
    const uint32_t j = qq / tk, lc = qq % tk;
    ac[((int64_t)b0 + j) * tk + lc] = (uint32_t)c;
    const int bit = ((r & 15) << 2) | (lc & 3);
    const int mine = (lc >> 2) * nbrow + (r >> 4);
    const uint64_t* pt = staged ? s_pt + j * nbk : gp + (int64_t)j * nbk;
    uint32_t nbr = 0, off = 0;
    for (int i = 0; i < nbk; ++i) {
      const uint64_t w = pt[i];
      nbr += w != 0ull;
      if (i < mine) off += __popcll(w);
    }
    off += __popcll(pt[mine] & ((1ull << bit) - 1ull));
    uint64_t vb;
    if (staged) {
      vb = s_vbase[j];
    } else {
      const uint32_t hdr = (nbc + 1 + nbr + 7) & ~7u;
      vb = sp[b0 + j] + hdr + 8 * nbr;
    }
    reinterpret_cast<float*>(packed + vb)[off] = v;
  }
  }  // panel loop
}

__global__ void k_finalize(const int64_t* __restrict__ rp, int64_t M, int64_t nnz, int64_t P,
                           const uint32_t* __restrict__ brp, const uint64_t* __restrict__ poff,
                           uint64_t* __restrict__ sp, const uint32_t* __restrict__ status,
                           uint64_t* __restrict__ info) {
  uint32_t st = *status;
  if (rp[0] != 0) st |= ST_RP0;
  if (rp[M] != nnz) st |= ST_NNZ;
  const uint64_t nb = brp[P];
  sp[nb] = poff[P];
  info[0] = nb;
  info[1] = poff[P];
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
  // panel lists: big (> kSmallCap, hub bitmap) | L1 (> kWarpCap) | L2 (CTA count) | L3 (CTA emit)
  uint32_t* biglist = (uint32_t*)dalloc(4 * (P + 1) * sizeof(uint32_t), s);
  uint32_t* l1 = biglist + (P + 1);
  uint32_t* l2 = biglist + 2 * (P + 1);
  uint32_t* l3 = biglist + 3 * (P + 1);
  uint32_t* ctr = (uint32_t*)dalloc(8 * sizeof(uint32_t), s);  // nbig, nl1, nl2, nl3, status
  const int64_t nparts = ceil_div(P + 1, kScanChunk) + 1;
  uint64_t* part = (uint64_t*)dalloc(nparts * sizeof(uint64_t), s);
  uint64_t* info = (uint64_t*)dalloc(4 * sizeof(uint64_t), s);  // [3] = status word | hub count
  const int big_ctas = num_sms();
  const int64_t words = ceil_div(K, 32) + 2;
  uint32_t* bigscr = (uint32_t*)dalloc((size_t)big_ctas * 2 * words * sizeof(uint32_t), s);
  hrpb_status_t st = HRPB_SUCCESS;
  if (!h->brp || !h->ac || !h->sp || !h->packed || !q || !cnt || !poff || !gpat || !biglist || !part || !info ||
      !bigscr || !ctr) {
    st = HRPB_ERROR_OUT_OF_MEMORY;
  }
  uint64_t hinfo[3] = {0, 0, 0};
  if (st == HRPB_SUCCESS) {
    uint32_t* nbig = ctr;
    uint32_t* nl1 = ctr + 1;
    uint32_t* nl2 = ctr + 2;
    uint32_t* nl3 = ctr + 3;
    uint32_t* status = ctr + 4;
    cudaMemsetAsync(ctr, 0, 8 * sizeof(uint32_t), s);
    const size_t count_smem =
        (size_t)kSmallCap * (8 + 4 + 4 + 1) + (size_t)ceil_div(kSmallCap, tk) * nbk * sizeof(uint64_t);
    const size_t wsm_c1 = (size_t)count_warp_smem<kWarpCap, true>(tm, tk) * kWarpsPerCta;
    const size_t wsm_c2 = (size_t)count_warp_smem<kWarpCap2, false>(tm, tk) * kWarpsPerCta;
    const size_t wsm_e1 = (size_t)emit_warp_smem<kWarpCap>(tm, tk) * kWarpsPerCta;
    const size_t wsm_e2 = (size_t)emit_warp_smem<kWarpCap2>(tm, tk) * kWarpsPerCta;
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_count_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_count_warp2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_emit_warp, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(k_emit_warp2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      attr = true;
    }
    const unsigned wgrid = (unsigned)ceil_div(P, kWarpsPerCta);
    const int mid_ctas = 8 * num_sms();
    if (P > 0) {  // pass A: warp (<= 256) -> warp, bitmap (<= 1024) -> CTA (<= 2048) -> hub bitmap
      k_count_warp<<<wgrid, 32 * kWarpsPerCta, wsm_c1, s>>>(row_ptr, col_idx, M, K, nnz, tm, tk, P, q, nact, nblk,
                                                            pbytes, gpat, l1, nl1, status);
      k_count_warp2<<<mid_ctas, 32 * kWarpsPerCta, wsm_c2, s>>>(row_ptr, col_idx, M, K, nnz, tm, tk, q, nact, nblk,
                                                                pbytes, gpat, l1, nl1, l2, nl2, l3, nl3, status);
      k_count<<<mid_ctas, kSmallThreads, count_smem, s>>>(row_ptr, col_idx, M, K, nnz, tm, tk, q, nact, nblk,
                                                          pbytes, gpat, l2, nl2, biglist, nbig, status);
      k_count_big<<<big_ctas, kBigThreads, 0, s>>>(row_ptr, col_idx, M, K, nnz, tm, tk, q, nact, nblk, pbytes, gpat,
                                                    biglist, nbig, bigscr, words, status);
      note_launch(4);
    }
    scan_excl<uint32_t>(nblk, P, h->brp, part, s);  // B2: blockedRowPtr
    scan_excl<uint64_t>(pbytes, P, poff, part, s);  // B4 (panel level): byte offset of each panel
    if (P > 0) {                                    // pass B
      k_emit_warp<<<wgrid, 32 * kWarpsPerCta, wsm_e1, s>>>(row_ptr, col_idx, values, M, K, nnz, tm, tk, P, q, nact,
                                                           h->brp, poff, gpat, h->ac, h->sp, h->packed);
      k_emit_warp2<<<mid_ctas, 32 * kWarpsPerCta, wsm_e2, s>>>(row_ptr, col_idx, values, M, K, nnz, tm, tk, q, nact,
                                                               h->brp, poff, gpat, h->ac, h->sp, h->packed, l1, nl1);
      k_emit<<<mid_ctas, kEmitThreads, 0, s>>>(row_ptr, col_idx, values, M, K, nnz, tm, tk, q, nact, h->brp, poff,
                                               gpat, h->ac, h->sp, h->packed, l3, nl3);
      note_launch(3);
    }
    k_finalize<<<1, 1, 0, s>>>(row_ptr, M, nnz, P, h->brp, poff, h->sp, status, info);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(hinfo, info, 3 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) st = cuda_status(e);
  }
  dfree(q, s); dfree(cnt, s); dfree(poff, s); dfree(gpat, s); dfree(biglist, s); dfree(part, s); dfree(info, s);
  dfree(bigscr, s);
  dfree(ctr, s);
  if (st == HRPB_SUCCESS && hinfo[2] != 0) st = HRPB_ERROR_INVALID_CSR;
  h->NB = (int64_t)hinfo[0];
  h->bytes = (int64_t)hinfo[1];
  return st;
}

}  // namespace hrpb
