// spmm_kernel.cuh — the hrpb_spmm_sm100 kernel template: C = A.B with A in HRPB.
//
// Paper kernel (Alg. "cuTeSpMM kernel design"; prose P:L244-282): one thread block
// per row panel, warps along N, SM_A/SM_B staging, per-brick pattern decode with prefix popcounts
// (P:L207-219), Ampere mma.sync m16n8k4 TF32 accumulating in registers.
//
// B200 design:
//  * persistent CTAs (one per SM), each owning a contiguous panel range balanced on
//    (blocks + panels) (S1);
//  * warps 0..3: producers — block i of the CTA goes to warp i % 4: cp.async.bulk of the packed block bytes (S2)
//    and cp.async 16-B copies of its TK gathered B rows (activeCols) into an MN-major SWIZZLE_128B_BASE32B tile;
//    the sentinel column K is zero-filled (S3) (TMA tile::gather4 staging as the GM = 0 variant);
//  * warps 4..7: decoders (block i -> warp 4 + i % 4) — prefix-popcount brick expansion into a
//    K-major TF32 tile (integer RNA rounding of A, reading R15) (S2);
//  * warps 8..9: one elected thread each issues tcgen05.mma.kind::tf32 computing the transposed product
//    D[n, r] += sum_k Bg[k, n] * A[r, k]  (M = 128 dense columns, N = TM panel rows, K = 8 x 2); block i of the
//    CTA goes to warp 8 + i % 2, which accumulates it into its own TMEM set of the panel's slot (S4);
//  * warps 12..15: epilogue — tcgen05.ld 32x32b of the panel's sets, summed, coalesced 128-B row stores (S5);
//  * mbarrier rings: full_a/full_b (TMA), dec (decoder), empty (tcgen05.commit), tfull/tempty.
#pragma once
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace hrpb {

constexpr int kProdWarps = 4;                              // warps 0..3: gather producers
constexpr int kDecWarps = 4;                               // warps 4..7: brick decoders
constexpr int kMmaWarp = kProdWarps + kDecWarps;           // warps 8..11: TMEM alloc (8) and MMA issue
constexpr int kMmaWarps = 4;                               // MMA-issuing warps (at most; SmemLayout::kMW are used)
constexpr int kEpiWarp0 = kMmaWarp + kMmaWarps;            // warps 12..15: epilogue (TMEM lane quadrant = warp % 4)
constexpr int kSpmmThreads = 32 * (kEpiWarp0 + 4);        // 512
constexpr int kMaxStages = 24;
#ifndef HRPB_L2PF
#define HRPB_L2PF 0
#endif
// experiment (off): L2 prefetch distance in own blocks — the producer bulk-prefetches the B rows of its block kL2Pf
// blocks ahead into L2 (cp.async.bulk.prefetch.L2, no shared memory held). Measured slower at every distance
// (2 / 4 / 8: c4 5.68 -> 8.3 / 10.0 / 10.0 ms, c2a TM = 64 0.247 -> 0.338 ms, c3 19.1 -> 19.4 ms): the prefetches
// queue in the same bulk-copy path as the A blocks
constexpr int kL2Pf = HRPB_L2PF;
#ifndef HRPB_AC_EF
#define HRPB_AC_EF 0
#endif
#ifndef HRPB_EPI_SLEEP
#define HRPB_EPI_SLEEP 0
#endif
#ifndef HRPB_L2PF_MODE
#define HRPB_L2PF_MODE 1  // 1: prefetch.global.L2 per 128-B line, 0: cp.async.bulk.prefetch.L2 per row
#endif
constexpr int kPfRing = 8 + kL2Pf;  // producer look-ahead ring in own blocks (x4 producer warps)

// NEXT-3: B row-sharded (hrpb_spmm_sharded). Shard r holds rows [r rps, min((r + 1) rps, K)) at ptr[r] (ld = ldb),
// local or peer-mapped (another GPU's memory over NVLink); the producer picks the shard per gathered row.
constexpr int kMaxShards = 32;
struct ShardDesc {
  const float* ptr[kMaxShards];
  uint32_t rps;  // rows per shard
  int nsh;
};
// per-call scratch of hrpb_spmm: split-panel workspace, its flag word and this call's epoch
struct Scratch {
  float* ws;
  uint64_t* flag;
  uint64_t epoch;
  uint64_t* ranges;  // [shares][4]: every S1 share's range (CtaWork), read by k_spmm_fixup
  const ShardDesc* sd = nullptr;  // GM = 2 launches only
  uint32_t nchunks = 0;   // dynamic S1: shares (0 = static, one share per CTA)
  uint32_t* ctr = nullptr;  // dynamic S1 claim counter
};
inline uint64_t next_epoch() {
  static std::atomic<uint64_t> e{0};
  return ++e;
}

struct SpmmParams {
  const uint32_t* brp;
  const uint32_t* ac;
  const uint64_t* sp;
  const uint8_t* packed;
  float* C;
  int64_t M, N, P, NB;
  int64_t p_lo, p_hi;  // panel range of this launch (the whole matrix, or one chunk of the pipelined host path)
  float* ws;           // split-panel partial tiles [G][2][TM][128 NT]
  uint64_t* split_flag;  // set to `epoch` by any CTA that writes a partial tile (k_spmm_fixup runs only then)
  uint64_t epoch;
  uint64_t* ranges;      // [G][4] CtaWork of every CTA: {pa, pb, bB | bE << 32, first_full | last_full << 1}
  const float* B;  // row-major K x ldb (cp.async gather mode)
  int64_t K, ldb;
  int n0;      // first output column of this launch
  int stages;  // pipeline depth
  long long* trace;  // optional: per-block event timestamps of CTA 0 (HRPB_TRACE), [6][kTraceN]
  // GM = 2 (row-sharded B): shard table (see ShardDesc); inv = 1 / rps for the shard estimate of a row
  const float* sh_ptr[kMaxShards];
  uint32_t sh_rps;
  float sh_inv;
  int nsh;
  uint32_t nchunks;     // 0: static S1 (CTA c takes share c of G); else dynamic: nchunks shares (ranges precomputed by
                        // k_spmm_chunks), CTA c starts with share c and then claims shares G, G + 1, ... in order
  uint32_t* chunk_ctr;  // claim counter (zeroed by k_spmm_chunks)
  const int32_t* row_map;  // NEXT-4: C row of each A row (hrpb_set_row_map), NULL = identity
  long long* cta_t;  // optional (HRPB_CTA_TIMES): per CTA {globaltimer at entry, at exit, blocks, panels}
  int debug;         // HRPB_DEBUG bits (experiments only): 1 = skip C stores, 2 = skip decode, 4 = skip MMA issue,
                     // 8 = skip A bulk copy, 16 = B gather zero-fill only (no global reads), 32 = no B cp.async at all
};
constexpr int kTraceN = 1024;
constexpr int kTraceSlots = 10;  // slot 8: per warp of CTA 0 {cycles waiting on mbarriers, cycles total};
                                 // slot 9: per CTA {cycles, blocks, panels, first panel}
// trace slots: 0 producer issue (after empty), 1 A arrived (decoder), 2 decode done, 3 B arrived (MMA),
//              4 MMA issued, 5 epilogue got tfull (per panel), 6 decoder slot table done, 7 decoder rows done
// Instrumentation (HRPB_TRACE timestamps, HRPB_DEBUG work-skipping bits) exists only in builds with
// -DHRPB_INSTRUMENT=1 (tools/build_variant.py); the product kernel carries none of it: the serial MMA/decoder
// loops are sensitive to every extra instruction.
#ifndef HRPB_INSTRUMENT
#define HRPB_INSTRUMENT 0
#endif
constexpr bool kInstr = HRPB_INSTRUMENT != 0;
#ifndef HRPB_EXP_SKIP
#define HRPB_EXP_SKIP 0  // experiments only: HRPB_DEBUG bits compiled in as constants (no instrumentation overhead)
#endif
__device__ __forceinline__ bool dbg(const SpmmParams& p, int bit) {
  return (HRPB_EXP_SKIP & bit) != 0 || (kInstr && (p.debug & bit));
}
__device__ __forceinline__ bool tracing(const SpmmParams& p) { return kInstr && p.trace != nullptr; }
__device__ __forceinline__ void trace_ev(const SpmmParams& p, int slot, uint32_t i) {
  if (tracing(p) && blockIdx.x == 0 && i < kTraceN) p.trace[slot * kTraceN + i] = clock64();
}
// mbarrier wait that accumulates the cycles spent waiting when tracing (role busy/idle breakdown)
__device__ __forceinline__ void mbar_wait_acc(const SpmmParams& p, uint64_t* bar, uint32_t parity, long long& acc) {
  if (tracing(p)) {
    const long long t0 = clock64();
    mbar_wait(bar, parity);
    acc += clock64() - t0;
  } else {
    mbar_wait(bar, parity);
  }
}

// instruction descriptor: D F32, A/B TF32, A MN-major, B K-major, N = TM (panel rows), M = 128
template <int TMV>
__host__ __device__ constexpr uint32_t idesc_tf32() {
  return (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (0u << 16) | ((uint32_t)(TMV >> 3) << 17) |
         ((128u >> 4) << 24);
}

template <int NT, int TMV, int TKV>
struct SmemLayout {
  static constexpr int kNA = 4 * NT;                 // 32-column atoms per 4-row group
  static constexpr int kBTile = TKV * 128 * 4 * NT;  // gathered rows per stage
  static constexpr int kNbc = TKV / 4;               // brick columns per block
  static constexpr int kNbrow = TMV / 16;            // brick rows per block
  static constexpr int kNbk = kNbc * kNbrow;         // brick slots per block
  static_assert(kNbk <= 32, "the decoder's slot table gives one lane per brick slot");
  // largest HRPB-v1 block: align8(5 + nbk) + 8 nbk + 4 TM TK, rounded to 128 B
  static constexpr int kARawBytes = ((((kNbc + 1 + kNbk + 7) & ~7) + 8 * kNbk + 4 * TMV * TKV) + 127) & ~127;
  static constexpr int kATileBytes = TMV * TKV * 4;  // TM x TK fp32 decoded block
  static constexpr int kLbo = TMV * 16;              // bytes between 4-column K groups of the decoded tile
  // decode in place (the tile overwrites its own raw block) when a lane holds all its items' values at once: the
  // stage then needs no separate tile (c2a at TM = 64: 12 -> 16 stages; the kernel is latency-bound on its ring)
  static constexpr int kItems = TMV * kNbc / 32;
  static constexpr bool kInPlace = kItems <= 8;
  static_assert(!kInPlace || kARawBytes >= kATileBytes, "the raw slot must hold the decoded tile");
  static constexpr int kStage = kBTile + kARawBytes + (kInPlace ? 0 : kATileBytes);
  // MMA issue is latency-bound per issuing thread (~50 cycles per tcgen05.mma, ~180 per tcgen05.commit, measured:
  // tools/microtests/umma_commit.cu), so kMW warps issue the blocks of a panel in turn (block i -> warp i % kMW),
  // each into its own accumulator set; the epilogue adds the sets. kMW = the most warps whose sets leave room for
  // two panels in flight in the 512 TMEM columns.
  static constexpr int kCols1 = NT * TMV;  // one accumulator set: TM columns per 128-column N tile
#ifndef HRPB_MW_MAX
#define HRPB_MW_MAX 2
#endif
#ifndef HRPB_MW_TM64
#define HRPB_MW_TM64 2
#endif
  static constexpr int kMWcap = TMV >= 64 ? HRPB_MW_TM64 : HRPB_MW_MAX;
  static constexpr int kMW = 2 * 4 * kCols1 <= 512 && kMWcap >= 4 ? 4 : (2 * 2 * kCols1 <= 512 && kMWcap >= 2 ? 2 : 1);
  static constexpr int kSetCols = kMW * kCols1;  // TMEM columns of one panel slot
  // TMEM accumulator slots (panels in flight between the MMA warps and the epilogue): 2 to 4
  static constexpr int kSlots = 512 / kSetCols < 4 ? 512 / kSetCols : 4;
  static_assert(kSlots >= 2, "two panel slots must fit in the 512 TMEM columns");
  static_assert(kMW <= kMmaWarps && kDecWarps % kMW == 0, "MMA warps");
  static constexpr int kSlotCols = kSlots * kSetCols;
  static constexpr uint32_t kTmemCols = kSlotCols <= 32 ? 32 : (kSlotCols <= 64 ? 64 : (kSlotCols <= 128 ? 128 : (kSlotCols <= 256 ? 256 : 512)));
};


// S1 work assignment. Work units: panel p owns units [brp[p] + w p, brp[p+1] + w (p + 1)), w = kPanelW — one per block plus w for
// its epilogue (so empty panels cost one unit). CTA c of G takes units [t_c, t_c+1) with t_c = c W / G snapped up
// to the next panel start unless the panel containing it is "big" (more than two whole CTA shares): such a panel
// is split between CTAs, each accumulating its blocks into a workspace tile, and k_spmm_fixup adds the partial
// tiles in CTA order (deterministic) into C.
// kPanelW: units per panel epilogue per 16 panel rows (the C store of TM rows), 1 = one block's worth
#ifndef HRPB_PANEL_W
#define HRPB_PANEL_W 5
#endif
constexpr uint64_t kPanelW = HRPB_PANEL_W;
// dynamic S1 (long launches): shares per SM, claimed in order by the persistent CTAs, and the nnz from which a launch
// counts as long (c3, 128M nnz, ~13 ms; c4 / c5 / c2a at <= 40M nnz are balanced by the static model)
#ifndef HRPB_DYN_SHARES
#define HRPB_DYN_SHARES 16
#endif
constexpr int kDynShares = HRPB_DYN_SHARES;
constexpr int kFixThreads = 512;  // k_spmm_fixup threads (one CTA per share boundary)
#ifndef HRPB_DYN_REV
#define HRPB_DYN_REV 1
#endif
// position in the matrix of the share claimed as number k (see k_spmm_chunks)
__host__ __device__ __forceinline__ uint32_t share_pos(uint32_t k, uint32_t n) { return HRPB_DYN_REV ? n - 1 - k : k; }
constexpr int64_t kDynMinNnz = 64ll << 20;
#ifndef HRPB_PANEL_W32
#define HRPB_PANEL_W32 5
#endif
#ifndef HRPB_PANEL_W64
#define HRPB_PANEL_W64 12
#endif
// measured on c3 (R-MAT, N = 256) with two MMA-issuing warps per panel: TM = 16 → 5 units (3 / 4 / 5 / 6 / 8:
// 16.0 / 14.4-14.8 / 13.7 / 13.9 / 14.9 ms), TM = 32 → 5 (3 / 5 / 8: 16.1 / 14.3 / 14.4 ms), TM = 64 → 12 (20: 15.7 ms);
// TM = 128 scales TM = 64's
template <int TMV>
__host__ __device__ constexpr uint64_t panel_weight() {
  return TMV == 16 ? kPanelW : TMV == 32 ? (uint64_t)HRPB_PANEL_W32 : TMV == 64 ? (uint64_t)HRPB_PANEL_W64
                                                                                : 2 * (uint64_t)HRPB_PANEL_W64;
}
template <uint64_t PW>
__device__ __forceinline__ uint64_t unit_of(const uint32_t* brp, int64_t p) {  // units before panel p
  return (uint64_t)brp[p] + PW * (uint64_t)p;
}
template <uint64_t PW>
__device__ __forceinline__ int64_t warp_panel_of_unit(const uint32_t* brp, int64_t lo, int64_t hi, uint64_t t) {
  // the same by a whole warp: 32-way search, ~log32(P) dependent loads instead of log2(P). Invariant: the answer
  // is in [lo, hi] (hi = none in [lo, hi)).
  const int lane = threadIdx.x & 31;
  while (hi - lo > 32) {
    const int64_t step = (hi - lo + 31) / 32;
    const int64_t idx = lo + lane * step;
    const bool pred = idx < hi && unit_of<PW>(brp, idx + 1) > t;
    const uint32_t m = __ballot_sync(0xffffffffu, pred);
    if (!m) {  // every probe <= t: the answer is past the last probe inside [lo, hi)
      const int64_t kmax = min((int64_t)31, (hi - 1 - lo) / step);
      lo = lo + kmax * step + 1;
      continue;
    }
    const int k = __ffs(m) - 1;  // f(lo + k step) > t, and f(lo + (k - 1) step) <= t when k > 0
    if (k == 0) return lo;
    const int64_t l0 = lo;
    lo = l0 + (int64_t)(k - 1) * step + 1;
    hi = l0 + (int64_t)k * step;  // (itself a candidate: "none in [lo, hi)" means hi)
  }
  const int64_t idx = lo + lane;
  const bool pred = idx < hi && unit_of<PW>(brp, idx + 1) > t;
  const uint32_t m = __ballot_sync(0xffffffffu, pred);
  return m ? lo + __ffs(m) - 1 : hi;
}
// boundary t_c and the panel containing unit t_c (p_hi if t_c is the end); FIND = (brp, lo, hi, t) -> panel
template <uint64_t PW, typename FIND>
__device__ __forceinline__ uint64_t work_boundary(const uint32_t* brp, int64_t p_lo, int64_t p_hi, uint64_t c,
                                                  uint64_t G, int64_t& pt, FIND find) {
  const uint64_t base = unit_of<PW>(brp, p_lo);
  const uint64_t W = unit_of<PW>(brp, p_hi) - base;
  if (c == 0) {
    pt = p_lo;
    return base;
  }
  if (c >= G) {
    pt = p_hi;
    return base + W;
  }
  const uint64_t t = base + c * W / G;
  const int64_t p = find(brp, p_lo, p_hi, t);
  pt = p;
  if (p >= p_hi) return base + W;
  const uint64_t start = unit_of<PW>(brp, p), end = unit_of<PW>(brp, p + 1);
  if (t == start) return t;
  // big panel (more than two whole CTA shares): split here. (At one share, launches with about one panel per CTA
  // split every larger-than-average panel, and the fix-up then costs more than the imbalance it removes.)
  if ((end - start) * G > 2 * W) return t;
  pt = p + 1;                               // small panel: round up to the next panel start
  return end;
}
struct CtaWork {
  int64_t pa, pb;      // panels [pa, pb) touched by this CTA (pb - 1 = pl, the panel of its last unit)
  uint32_t bB, bE;     // its flat block range
  bool first_full, last_full;  // owns all units of pa / of pb - 1
};
// the share between boundaries f0 < f1 of a grid of G equal shares (cta_work: f0 = c, f1 = c + 1)
template <uint64_t PW, typename FIND>
__device__ __forceinline__ CtaWork cta_work_span(const uint32_t* brp, int64_t p_lo, int64_t p_hi, uint64_t f0,
                                                 uint64_t f1, uint64_t G, FIND find) {
  CtaWork w;
  int64_t p0, p1;
  const uint64_t t0 = work_boundary<PW>(brp, p_lo, p_hi, f0, G, p0, find);
  const uint64_t t1 = work_boundary<PW>(brp, p_lo, p_hi, f1, G, p1, find);
  if (t1 <= t0) {
    w.pa = w.pb = p_lo;
    w.bB = w.bE = brp[p_lo];
    w.first_full = w.last_full = true;
    return w;
  }
  w.pa = p0;  // the panel containing unit t0
  // the panel containing unit t1 - 1: p1 unless t1 is exactly p1's first unit (then the one before)
  const int64_t pl = (p1 >= p_hi || t1 == unit_of<PW>(brp, p1)) ? p1 - 1 : p1;
  w.pb = pl + 1;
  w.first_full = t0 == unit_of<PW>(brp, w.pa);
  w.last_full = t1 == unit_of<PW>(brp, pl + 1);
  // (a boundary inside a panel's epilogue units maps past its last block: clamp to the panel's blocks)
  w.bB = (uint32_t)max((uint64_t)brp[w.pa], min((uint64_t)brp[w.pa + 1], t0 - PW * (uint64_t)w.pa));
  w.bE = (uint32_t)min((uint64_t)brp[pl + 1], t1 - PW * (uint64_t)pl);
  if (!w.first_full && w.bB >= brp[w.pa + 1]) {
    // the range starts inside a split panel's epilogue units: it owns none of that panel's blocks (the fix-up
    // stores the panel), so its first panel is the next one, from its start (else this CTA would treat the
    // panel as one with no blocks and zero-fill its C rows)
    ++w.pa;
    w.first_full = true;
    w.bB = brp[w.pa];
    if (w.pa >= w.pb) {
      w.pb = w.pa;
      w.bE = w.bB;
    }
  }
  return w;
}
template <uint64_t PW, typename FIND>
__device__ __forceinline__ CtaWork cta_work(const uint32_t* brp, int64_t p_lo, int64_t p_hi, uint64_t c, uint64_t G,
                                            FIND find) {
  return cta_work_span<PW>(brp, p_lo, p_hi, c, c + 1, G, find);
}
template <uint64_t PW>
struct WarpFind {
  __device__ int64_t operator()(const uint32_t* b, int64_t lo, int64_t hi, uint64_t t) const {
    return warp_panel_of_unit<PW>(b, lo, hi, t);
  }
};

// Warp-cooperative iteration over panels [pa, pb): blockedRowPtr is fetched 32 panels per coalesced
// load, one chunk ahead. All 32 lanes must call next() convergently; it returns false at the end.
struct PanelCursor {
  const uint32_t* brp;
  int64_t pb, base, j;
  int cnt;
  uint32_t cur, cur_last, nxt, nxt_last;
  int lane;
  __device__ void load(int64_t b0, uint32_t& v, uint32_t& last) {
    const int64_t idx = b0 + lane;
    v = idx <= pb ? __ldg(brp + idx) : 0u;
    last = __ldg(brp + (b0 + 32 <= pb ? b0 + 32 : pb));
  }
  __device__ PanelCursor(const uint32_t* brp_, int64_t pa, int64_t pb_, int lane_)
      : brp(brp_), pb(pb_), base(pa), j(-1), lane(lane_) {
    cnt = (int)min((int64_t)32, pb - pa);
    if (pa < pb) load(pa, cur, cur_last);
    if (pa + 32 < pb) load(pa + 32, nxt, nxt_last);
  }
  // advances to the next panel; p = panel id, bb/be = its block range
  __device__ bool next(int64_t& p, uint32_t& bb, uint32_t& be) {
    if (base >= pb) return false;
    if (++j == cnt) {
      base += 32;
      if (base >= pb) return false;
      cur = nxt;
      cur_last = nxt_last;
      cnt = (int)min((int64_t)32, pb - base);
      j = 0;
      if (base + 32 < pb) load(base + 32, nxt, nxt_last);
    }
    p = base + j;
    bb = __shfl_sync(0xffffffffu, cur, (int)j);
    const uint32_t nx = __shfl_sync(0xffffffffu, cur, (int)(j + 1) & 31);
    be = j + 1 < 32 ? nx : cur_last;
    return true;
  }
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_async16_hint(uint32_t dst, const void* src, uint32_t src_bytes, uint64_t pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(dst), "l"(src), "r"(src_bytes),
               "l"(pol) : "memory");
}
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {  // bytes: multiple of 16
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// GM = gather mode: 0 = TMA tile::gather4 (one issuing lane per producer warp),
//                   1 = cp.async 16-B copies by all 128 producer threads into the same swizzled layout.
// DYN: dynamic S1 shares (a separate instantiation: the share loop costs the static kernel registers and time);
// RMAP: C rows through the handle's row map (NEXT-4; separate for the same reason: c2b 0.172 -> 0.207 ms)
template <int NT, int GM, int TMV, int TKV, bool DYN = false, bool RMAP = false>
__global__ void __launch_bounds__(kSpmmThreads, 1) k_spmm(const __grid_constant__ CUtensorMap tmB,
                                                    const __grid_constant__ SpmmParams prm) {
  pdl_wait();
  constexpr uint64_t kPW = panel_weight<TMV>();  // S1 units per panel epilogue
  using L = SmemLayout<NT, TMV, TKV>;
  static_assert(GM != 0 || TKV == 16, "TMA gather4 staging is written for TK = 16");
  constexpr int kARawBytes = L::kARawBytes, kATileBytes = L::kATileBytes;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // 1024-B alignment by pointer arithmetic on the __shared__ array (an integer round trip would make every
  // derived pointer generic: LD.E/ST.E instead of LDS/STS)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const int S = prm.stages;
  uint8_t* btile0 = smem;                                 // S x kBTile (1024-aligned)
  uint8_t* araw0 = smem + (size_t)S * L::kBTile;          // S x kARawBytes
  uint8_t* atile0 = L::kInPlace ? araw0 : araw0 + (size_t)S * kARawBytes;  // decoded tiles (in place: the raw slots)
  constexpr int kATileStride = L::kInPlace ? kARawBytes : kATileBytes;
  uint64_t* bars = (uint64_t*)(araw0 + (size_t)S * kARawBytes + (L::kInPlace ? 0 : (size_t)S * kATileBytes));
  uint64_t* full_a = bars;
  uint64_t* full_b = bars + S;
  uint64_t* empty = bars + 2 * S;
  uint64_t* tfull = bars + 3 * S;
  uint64_t* tempty = tfull + 4;
  uint32_t* misc = (uint32_t*)(tempty + 4);  // [0] tmem base
  int64_t* range = (int64_t*)(misc + 2);     // CtaWork: pa, pb, bB, bE, first_full, last_full
  // per decoder warp: brick-slot table (pattern, value offset) of the block being decoded
  uint64_t* slot_pat = (uint64_t*)(range + 6);                 // [kDecWarps][kNbk]
  uint32_t* slot_off = (uint32_t*)(slot_pat + kDecWarps * L::kNbk);  // [kDecWarps][kNbk]
  // per producer warp: ring of kPfRing own blocks {sizePtr[b], sizePtr[b + 1], activeCols[b * TK .. + TK)}
  uint32_t* pring = (uint32_t*)(((uintptr_t)(slot_off + kDecWarps * L::kNbk) + 15) & ~(uintptr_t)15);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  long long wacc = 0;
  if (prm.cta_t && tid == 0) prm.cta_t[4 * blockIdx.x] = (long long)globaltimer();
  const long long t_start = kInstr ? clock64() : 0;
  const uint32_t tmem_cols = L::kTmemCols;

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_a[s], 1);
      // B rows landed (one producer warp per block: 1 expect_tx arrive or 32 cp.async noinc arrivals) AND the
      // block's A tile is decoded (+1 decoder arrival): the MMA warp waits on this single barrier per block
      mbar_init(&full_b[s], (GM == 0 ? 1 : 32) + 1);  // (GM 1, 2: cp.async)
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < L::kSlots; ++i) { mbar_init(&tfull[i], L::kMW); mbar_init(&tempty[i], 4); }
    fence_mbar_init();

    prefetch_tmap(&tmB);
  }
  if (warp == kMmaWarp) tmem_alloc(&misc[0], tmem_cols);
  const uint32_t* __restrict__ brp = prm.brp;
  const int n0 = prm.n0;
  const int64_t N = prm.N, M = prm.M;
  uint32_t tbase = 0;
  // running state across this CTA's shares (dynamic S1): blocks of earlier shares (the block index that picks
  // stages, parities and the MMA warp continues), and the panel counters of the MMA warps and the epilogue (TMEM
  // slot sequence)
  uint32_t base = 0, pc_mma = 0, pc_epi = 0;
  uint32_t chunk = blockIdx.x;
  for (;;) {
  if (warp == 0) {  // S1: contiguous range of ~equal work (blocks + panels) in [p_lo, p_hi); big panels may split
    if (!DYN) {
      const CtaWork cw = cta_work<kPW>(prm.brp, prm.p_lo, prm.p_hi, blockIdx.x, gridDim.x, WarpFind<kPW>());
      if (lane == 0) {
        range[0] = cw.pa; range[1] = cw.pb; range[2] = cw.bB; range[3] = cw.bE;
        range[4] = cw.first_full; range[5] = cw.last_full;
        if (cw.bB < cw.bE && !(cw.first_full && cw.last_full)) *prm.split_flag = prm.epoch;
        uint64_t* rg = prm.ranges + 4 * blockIdx.x;  // (the fix-up reads the ranges instead of re-deriving them)
        rg[0] = (uint64_t)cw.pa;
        rg[1] = (uint64_t)cw.pb;
        rg[2] = (uint64_t)cw.bB | ((uint64_t)cw.bE << 32);
        rg[3] = (uint64_t)cw.first_full | ((uint64_t)cw.last_full << 1);
      }
    } else if (lane == 0) {  // the share's range, precomputed by k_spmm_chunks
      const uint64_t* rg = prm.ranges + 4 * (size_t)share_pos(chunk, prm.nchunks);
      range[0] = (int64_t)rg[0]; range[1] = (int64_t)rg[1];
      range[2] = (int64_t)(uint32_t)rg[2]; range[3] = (int64_t)(rg[2] >> 32);
      range[4] = (int64_t)(rg[3] & 1); range[5] = (int64_t)((rg[3] >> 1) & 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  tbase = misc[0];
  const int64_t pa = range[0], pb = range[1];
  const uint32_t cbB = (uint32_t)range[2], cbE = (uint32_t)range[3];
  const bool first_full = range[4] != 0, last_full = range[5] != 0;

  if (warp < kProdWarps) {
    // ---------------------------------------------------------------- producers (warps 0..3)
    // Warp w stages blocks i = w, w+4, ... (the i-th block of this CTA uses stage i % S): the packed
    // block bytes (S2, one bulk copy) and its 16 gathered B rows (S3). One cp.async instruction moves one
    // contiguous 512-B row segment (lane = 16-B chunk); lanes 0..15 prefetch the block's activeCols 8 blocks
    // ahead and the row index is broadcast by shuffle.
    const uint64_t pol_a = policy_evict_first();
#ifdef HRPB_HOT_EXP
    uint64_t pol_hot, pol_cold = pol_a;
#if HRPB_HOT_POL == 0
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol_hot));
#elif HRPB_HOT_POL == 1
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_hot));
#else
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 0.5;" : "=l"(pol_hot));
#endif
#endif
    const int na_eff = (int)min((int64_t)L::kNA, ceil_div(N - n0, 32));  // 32-col atoms with a column < N
    const int64_t b_begin = cbB, b_end = cbE;
    const int pw = warp;
    const uint32_t Kr = (uint32_t)prm.K;
    const int64_t ldb = prm.ldb;
    const float* __restrict__ Bsrc = prm.B + n0;
    const uint32_t* __restrict__ acp = prm.ac;
    const uint64_t* __restrict__ spp = prm.sp;
    const uint8_t* __restrict__ pk = prm.packed;
    const int row = lane & (TKV - 1);
    const uint32_t bt0 = smem_u32(btile0);
    const uint32_t ldb32 = (uint32_t)ldb;                       // (N < 2^31)
    const float* __restrict__ Blane = Bsrc + 4 * lane;
    // Look-ahead ring in shared memory, filled with cp.async (4-B activeCols rows, 8-B sizePtr pairs) kPfRing own
    // blocks ahead and committed as one cp.async group per block: waiting for the group of block b
    // (wait_group kPfRing - 1) never waits on a load issued in the same iteration, and a register ring would
    // stall on the moves of its in-flight loads. The block loop is not unrolled (code size: the kernel's roles
    // share the instruction cache).
    constexpr int kSlotW = TKV + 4;  // words per ring slot: sp pair (4 words) + TK rows
    uint32_t* myring = pring + pw * kPfRing * kSlotW;
    auto fetch = [&](int64_t bl, int q) {  // stage block bl's look-ahead data into ring slot q (all lanes call)
      uint32_t* slot = myring + q * kSlotW;
      if (bl < b_end) {
#if HRPB_AC_EF  // experiment: activeCols / sizePtr (streamed once) with the L2 evict-first policy
        if (lane < TKV)
          asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 4, %2;" ::"r"(smem_u32(slot + 4 + lane)),
                       "l"(acp + bl * TKV + lane), "l"(pol_a) : "memory");
        if (lane < 2)
          asm volatile("cp.async.ca.shared.global.L2::cache_hint [%0], [%1], 8, %2;" ::"r"(smem_u32(slot + 2 * lane)),
                       "l"(spp + bl + lane), "l"(pol_a) : "memory");
#else
        if (lane < TKV)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(slot + 4 + lane)),
                       "l"(acp + bl * TKV + lane) : "memory");
        if (lane < 2)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(slot + 2 * lane)),
                       "l"(spp + bl + lane) : "memory");
#endif
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // lane-constant destination offsets (per 128-column tile t and row % 4) and column bounds
    uint32_t doff[NT][4];
    bool col_ok[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int c = lane + 32 * t;  // 16-B chunk along N
      const int at = c >> 3;
      const uint32_t g = (c >> 1) & 3;
#pragma unroll
      for (int rq = 0; rq < 4; ++rq) doff[t][rq] = at * 512 + ((g ^ rq) << 5) + ((c & 1) << 4);
      col_ok[t] = (n0 + 4 * c) < N && at < na_eff;
    }
    const uint32_t i0p = base + (uint32_t)pw;  // running block index of this warp's first block of the share
    int s = (int)(i0p % (uint32_t)S);
    uint32_t ph = (i0p / (uint32_t)S) & 1u;
    int64_t b = b_begin + pw;
#pragma unroll
    for (int q = 0; q < kPfRing; ++q) fetch(b + 4 * q, q);
    int q = 0;
    // prefetched row segment: this CTA's columns [n0, n0 + 128 NT) of a B row, whole 16-B chunks only
    const int64_t pf_cols = min((int64_t)(128 * NT), prm.N - n0);
    const uint32_t pf_bytes = (uint32_t)((pf_cols * 4) & ~15ll);
#pragma unroll 1
    for (; b < b_end; b += 4) {
      // the groups of blocks b .. b + 4 kL2Pf are complete (one group per block, kPfRing committed ahead)
      asm volatile("cp.async.wait_group %0;" ::"n"(kPfRing - 1 - kL2Pf) : "memory");
      __syncwarp();
      const uint32_t* slot = myring + q * kSlotW;
      if constexpr (kL2Pf > 0) {
        const int qp = q + kL2Pf < kPfRing ? q + kL2Pf : q + kL2Pf - kPfRing;
        if (b + 4 * kL2Pf < b_end && pf_bytes) {
#if HRPB_L2PF_MODE == 1
          // per-lane prefetch.global.L2 of the 128-B lines of the TK rows (LSU path, no shared memory held)
          const uint32_t lines = (pf_bytes + 127) >> 7;
          for (uint32_t x = lane; x < TKV * lines; x += 32) {
            const uint32_t rw = x / lines, ln = x - rw * lines;
            const uint32_t rk = myring[qp * kSlotW + 4 + rw];
            if (rk < Kr) asm volatile("prefetch.global.L2 [%0];" ::"l"(Bsrc + (uint64_t)rk * ldb32 + 32 * ln));
          }
#else
          if (lane < TKV) {
            const uint32_t rk = myring[qp * kSlotW + 4 + lane];
            if (rk < Kr) prefetch_l2_bulk(Bsrc + (uint64_t)rk * ldb32, pf_bytes);
          }
#endif
        }
      }
      mbar_wait_acc(prm, &empty[s], ph ^ 1, wacc);
      if (lane == 0) {
        trace_ev(prm, 0, (uint32_t)(b - b_begin));
        const uint64_t s0 = *reinterpret_cast<const uint64_t*>(slot), s1 = *reinterpret_cast<const uint64_t*>(slot + 2);
        const uint32_t a_bytes = (uint32_t)(s1 - s0);
        if (dbg(prm, 8)) {
          mbar_arrive(&full_a[s]);
        } else {
          mbar_expect_tx(&full_a[s], a_bytes);
          bulk_g2s(araw0 + (size_t)s * kARawBytes, pk + s0, a_bytes, &full_a[s], pol_a);
        }
      }
      const uint32_t bt = bt0 + s * L::kBTile;
      uint32_t rr[TKV];
#pragma unroll
      for (int k4 = 0; k4 < TKV / 4; ++k4) {
        const uint4 v4 = *reinterpret_cast<const uint4*>(slot + 4 + 4 * k4);
        rr[4 * k4] = v4.x; rr[4 * k4 + 1] = v4.y; rr[4 * k4 + 2] = v4.z; rr[4 * k4 + 3] = v4.w;
      }
      if constexpr (GM == 0) {
        if (lane == 0) {
          mbar_expect_tx(&full_b[s], 16u * 128u * (uint32_t)na_eff);
          uint8_t* btg = btile0 + (size_t)s * L::kBTile;
#pragma unroll
          for (int g4 = 0; g4 < 4; ++g4)
            for (int a = 0; a < na_eff; ++a)
              tma_gather4(btg + (g4 * L::kNA + a) * 512, &tmB, n0 + 32 * a, (int32_t)rr[4 * g4],
                          (int32_t)rr[4 * g4 + 1], (int32_t)rr[4 * g4 + 2], (int32_t)rr[4 * g4 + 3], &full_b[s]);
        }
      } else {
        // lane copies 16-B chunk c = lane + 32 t (along N) of each of the TK rows; destination in the UMMA
        // SWIZZLE_128B_BASE32B MN-major atom: 4 rows x 128 B, 32-B granule g stored at g ^ (row % 4).
#pragma unroll
        for (int rw = 0; rw < TKV; ++rw) {
          if (dbg(prm, 32)) break;
          const uint32_t rk = rr[rw];
          const bool real = rk < Kr && !(dbg(prm, 16));  // sentinel K -> zero fill (src-size 0)
          const float* src;
          if constexpr (GM == 2) {  // row-sharded B: shard r = rk / rps (float estimate, corrected by one step)
            const uint32_t rq = real ? rk : 0u, rps = prm.sh_rps;
            uint32_t r = __float2uint_rz(__uint2float_rz(rq) * prm.sh_inv);
            r = min(r, (uint32_t)prm.nsh - 1u);
            if (rq < r * rps) --r;
            else if (r + 1u < (uint32_t)prm.nsh && rq >= (r + 1u) * rps) ++r;
            src = prm.sh_ptr[r] + n0 + 4 * lane + (uint64_t)(rq - r * rps) * ldb32;
          } else {
            src = Blane + (uint64_t)(real ? rk : 0u) * ldb32;
          }
          const uint32_t rowb = bt + (rw >> 2) * (L::kNA * 512) + (rw & 3) * 128;
#ifdef HRPB_HOT_EXP  // experiment: L2 priority by an R-MAT popularity proxy (few one bits in the id)
          const uint64_t pol = __popc(rk) <= HRPB_HOT_EXP ? pol_hot : pol_cold;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (t * 4 < na_eff)
              cp_async16_hint(rowb + doff[t][rw & 3], src + 128 * t, (real && col_ok[t]) ? 16u : 0u, pol);
          }
#else
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            if (t * 4 < na_eff) cp_async16(rowb + doff[t][rw & 3], src + 128 * t, (real && col_ok[t]) ? 16u : 0u);
          }
#endif
        }
        if (dbg(prm, 32)) mbar_arrive(&full_b[s]);
        else cp_async_arrive_noinc(&full_b[s]);
      }
      __syncwarp();  // every lane has read slot q before it is refilled
      fetch(b + 4 * kPfRing, q);
      q = q + 1 == kPfRing ? 0 : q + 1;
      s += 4;
      if (s >= S) { s -= S; ph ^= 1; }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");  // (the look-ahead groups past the share's end)
  } else if (warp < kMmaWarp) {
    // ---------------------------------------------------------------- decoders (block i -> warp 4 + i % 4)
    // Lane l expands bits l and l+32 of each brick. All four patterns are loaded first, then
    // the values, so the per-block latency is ~3 dependent shared loads.
    const int dw = warp - kProdWarps;
    const int64_t b_begin = cbB, b_end = cbE;
    const uint32_t nib_sh = (uint32_t)(lane & 15) * 4u;            // tile row r with r % 16 == lane % 16
    const uint64_t below_row = (1ull << nib_sh) - 1ull;            // pattern bits of the rows above it
    const uint32_t i0d = base + (uint32_t)dw;
    int s = (int)(i0d % (uint32_t)S);
    uint32_t ph = (i0d / (uint32_t)S) & 1u;
    for (int64_t b = b_begin + dw; b < b_end; b += kDecWarps) {
      mbar_wait_acc(prm, &full_a[s], ph, wacc);
      if (lane == 0) trace_ev(prm, 1, (uint32_t)(b - b_begin));
      if (dbg(prm, 2)) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&full_b[s]);
        s += kDecWarps;
        if (s >= S) { s -= S; ph ^= 1; }
        continue;
      }
      const uint8_t* blk = araw0 + (size_t)s * kARawBytes;
      float* tile = reinterpret_cast<float*>(atile0 + (size_t)s * kATileStride);
      const uint64_t cp = *reinterpret_cast<const uint64_t*>(blk);  // colPtr[0..7] (bytes)
      const uint32_t nbr = blk[L::kNbc];                            // colPtr[nbc] = stored bricks
      const uint32_t hdr = (L::kNbc + 1 + nbr + 7) & ~7u;
      const uint64_t* pats = reinterpret_cast<const uint64_t*>(blk + hdr);
      const float* vals = reinterpret_cast<const float*>(blk + hdr + 8 * nbr);
      // (1) slot table: lane k < nbr owns stored brick k (CSC order); value offset = exclusive scan of popcounts
      uint64_t* tpat = slot_pat + dw * L::kNbk;
      uint32_t* toff = slot_off + dw * L::kNbk;
      if (lane < L::kNbk) {  // absent bricks: pattern 0, offset 0 (their loads below stay in bounds)
        tpat[lane] = 0ull;
        toff[lane] = 0u;
      }
      __syncwarp();
      uint64_t mypat = 0ull;
      uint32_t mycnt = 0, myslot = 0;
      if ((uint32_t)lane < nbr) {
        mypat = pats[lane];
        uint32_t bc = 0;
#pragma unroll
        for (int c = 1; c < L::kNbc; ++c) bc += (uint32_t)lane >= (uint32_t)((cp >> (8 * c)) & 0xFF);
        myslot = bc * L::kNbrow + (L::kNbrow == 1 ? 0u : (uint32_t)blk[L::kNbc + 1 + lane]);
        mycnt = __popcll(mypat);
      }
      uint32_t incl = mycnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if ((uint32_t)lane < nbr) {
        tpat[myslot] = mypat;
        toff[myslot] = incl - mycnt;
      }
      __syncwarp();
      if (lane == 0) trace_ev(prm, 6, (uint32_t)(b - b_begin));
      // (2) item q = lane + 32 j (j < TM/8) is (tile row r = q % TM, brick column bc = q / TM): the row's 4-bit
      // nibble of the brick pattern selects up to 4 values at prefix-popcount ranks; one 16-B store
      // per item into the K-major tile. Branch-free: every item's loads are issued before any is consumed, so a
      // block costs ~3 dependent shared-memory round trips (a divergent per-item branch serialised them).
      constexpr int kItems = L::kItems;
      constexpr int kChunk = kItems < 8 ? kItems : 8;  // items in flight per lane (all of them when in place)
      const uint32_t* __restrict__ uvals = reinterpret_cast<const uint32_t*>(vals);
#pragma unroll
      for (int j0 = 0; j0 < kItems; j0 += kChunk) {
        uint64_t ipat[kChunk];
        uint32_t ioff[kChunk];
#pragma unroll
        for (int jj = 0; jj < kChunk; ++jj) {
          const int q = lane + 32 * (j0 + jj), r = q % TMV, bc = q / TMV;
          const int slot = bc * L::kNbrow + (r >> 4);
          ipat[jj] = tpat[slot];
          ioff[jj] = toff[slot];
        }
        uint4 iv[kChunk];
        uint32_t inib[kChunk];
#pragma unroll
        for (int jj = 0; jj < kChunk; ++jj) {
          // row r % 16 == lane % 16 for every item of this lane: the nibble shift and the below-mask are constant
          const uint32_t nib = (uint32_t)(ipat[jj] >> nib_sh) & 0xFu;
          const uint32_t i0 = ioff[jj] + (uint32_t)__popcll(ipat[jj] & below_row);
          const uint32_t i1 = i0 + (nib & 1u), i2 = i1 + ((nib >> 1) & 1u), i3 = i2 + ((nib >> 2) & 1u);
          // unselected lanes read at most 3 words past the block's values: still inside the stage ring
          iv[jj] = make_uint4(uvals[i0], uvals[i1], uvals[i2], uvals[i3]);
          inib[jj] = nib;
        }
        if constexpr (L::kInPlace) __syncwarp();  // every lane has read the raw block before the tile overwrites it
#pragma unroll
        for (int jj = 0; jj < kChunk; ++jj) {
          const int q = lane + 32 * (j0 + jj), r = q % TMV, bc = q / TMV;
          const uint32_t nib = inib[jj];
          // FP32 -> TF32 round-to-nearest (ties away) as integer ops, value kept only where the pattern bit is set
          // (reading R15; cvt.rna.tf32.f32 is a ~7-instruction emulation on sm_100a). Finite A assumed (R17).
          uint4 v;
          v.x = (iv[jj].x + 0x1000u) & ((nib & 1u) ? 0xFFFFE000u : 0u);
          v.y = (iv[jj].y + 0x1000u) & ((nib & 2u) ? 0xFFFFE000u : 0u);
          v.z = (iv[jj].z + 0x1000u) & ((nib & 4u) ? 0xFFFFE000u : 0u);
          v.w = (iv[jj].w + 0x1000u) & ((nib & 8u) ? 0xFFFFE000u : 0u);
          *reinterpret_cast<uint4*>(tile + bc * (L::kLbo / 4) + (r >> 4) * 64 + (r & 15) * 4) = v;
        }
      }
      if (lane == 0) trace_ev(prm, 7, (uint32_t)(b - b_begin));
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        trace_ev(prm, 2, (uint32_t)(b - b_begin));
        mbar_arrive(&full_b[s]);
      }
      s += kDecWarps;
      if (s >= S) { s -= S; ph ^= 1; }
    }
  } else if (warp < kEpiWarp0) {
    // ---------------------------------------------------------------- MMA issuers (one thread per warp)
    // Block i of this CTA's range goes to MMA warp i % kMW (the decoders' and producers' interleave), which
    // accumulates it into its own TMEM set of the panel's slot (pc % kSlots): the issue latency of one thread
    // (~50 cycles per tcgen05.mma, ~180 per tcgen05.commit) no longer serialises a long panel. Every MMA warp walks
    // every panel that has blocks here: it waits for the slot to be free, issues its blocks (if any) and commits
    // (or, with none, plain-arrives) on tfull[slot] (kMW arrivals). Stage j % S is only ever consumed by warp
    // j % kMW (S is a multiple of 4), in order, so its parity (j / S) & 1 is unambiguous.
    constexpr int kMW = L::kMW;
    const int mw = warp - kMmaWarp;
    if (mw < kMW) {
      const int64_t b_begin = cbB;
      uint32_t pc = pc_mma;
      constexpr uint32_t kIdesc = idesc_tf32<TMV>();
      // descriptors of stage 0; stage s adds s * stage bytes / 16 to the start-address field (no carry: < 256 KB)
      const uint64_t adesc0 = umma_sdesc(smem_u32(btile0), 512, L::kNA * 512, 1);
      const uint64_t bdesc0 = umma_sdesc(smem_u32(atile0), L::kLbo, 128, 0);
      const uint32_t Su = (uint32_t)S;
      PanelCursor cursor(brp, pa, pb, lane);
      int64_t p;
      uint32_t bb, be;
      while (cursor.next(p, bb, be)) {
        bb = bb > cbB ? bb : cbB;  // this CTA's blocks of the panel (all of them unless the panel is split)
        be = be < cbE ? be : cbE;
        if (bb >= be) continue;
        const uint32_t slot = pc % L::kSlots;
        // running block range of the panel here (the index continues across this CTA's shares)
        const uint32_t i0 = base + (uint32_t)(bb - b_begin), i1 = base + (uint32_t)(be - b_begin);
        const uint32_t j0 = i0 + (((uint32_t)mw + kMW - i0 % kMW) % kMW);              // first own block
        mbar_wait_acc(prm, &tempty[slot], ((pc / L::kSlots) & 1) ^ 1, wacc);
        tc_fence_after();
        const uint32_t dcol = tbase + slot * L::kSetCols + mw * L::kCols1;
        for (uint32_t j = j0; j < i1; j += kMW) {
          const uint32_t st = j % Su, ph = (j / Su) & 1u;
          mbar_wait_acc(prm, &full_b[st], ph, wacc);
          tc_fence_after();
          if (lane == 0) {
            trace_ev(prm, 3, j);
            trace_ev(prm, 4, j);
            if (dbg(prm, 4)) {
              mbar_arrive(&empty[st]);
            } else {
              const uint64_t ad = adesc0 + (uint64_t)(st * (uint32_t)(L::kBTile >> 4));
              const uint64_t bd = bdesc0 + (uint64_t)(st * (uint32_t)(kATileStride >> 4));
              // K step outer, N tile inner: consecutive MMAs write different accumulators (independent)
#pragma unroll
              for (int g = 0; g < TKV / 8; ++g) {
#pragma unroll
                for (int t = 0; t < NT; ++t)
                  umma_tf32(dcol + t * TMV, ad + (uint64_t)(((2 * g * L::kNA + 4 * t) * 512) >> 4),
                            bd + (uint64_t)((g * 2 * L::kLbo) >> 4), kIdesc, (j > j0 || g > 0) ? 1u : 0u);
              }
              umma_commit(&empty[st]);
            }
          }
          __syncwarp();
        }
        if (lane == 0) {
          if (j0 < i1) umma_commit(&tfull[slot]);
          else mbar_arrive(&tfull[slot]);  // no block of this panel here: its set is not read
        }
        __syncwarp();
        ++pc;
      }
      pc_mma = pc;
    }
  } else {
    // ---------------------------------------------------------------- epilogue (last 4 warps)
    const int qd = warp & 3;            // TMEM lane quadrant accessible to this warp
    const int et = tid - 32 * kEpiWarp0;  // 0..127
    const int64_t ncols = min((int64_t)128 * NT, N - n0);
    uint32_t pc = pc_epi;
    PanelCursor cursor(brp, pa, pb, lane);
    int64_t p;
    uint32_t bb, be;
    while (cursor.next(p, bb, be)) {
      const int64_t row0 = p * TMV;
      const int nrows = (int)min((int64_t)TMV, M - row0);
      if (bb == be) {  // empty panel (always owned whole): zero rows (R13)
        for (int r = 0; r < nrows; ++r) {
          const int64_t cr = RMAP ? (int64_t)prm.row_map[row0 + r] : row0 + r;
          for (int64_t c = et; c < ncols; c += 128) prm.C[cr * N + n0 + c] = 0.f;
        }
        continue;
      }
      const bool full = (p != pa || first_full) && (p != pb - 1 || last_full);
      const uint32_t cb = bb > cbB ? bb : cbB, ce = be < cbE ? be : cbE;
      if (cb >= ce) continue;  // split panel without blocks here
      // accumulator sets written: MMA warp w took the blocks i = w (mod kMW) of the CTA-local range [i0, i0 + n)
      constexpr int kMW = L::kMW;
      const uint32_t i0 = base + (cb - cbB), nblk = ce - cb;
      uint32_t cmask = 0;
#pragma unroll
      for (int w = 0; w < kMW; ++w)
        if (nblk >= (uint32_t)kMW || ((uint32_t)w + kMW - i0 % kMW) % kMW < nblk) cmask |= 1u << w;
      // a split panel's share goes to this CTA's workspace tile (slot 0: its first panel, 1: its last)
      float* const obase = full ? prm.C + row0 * N + n0
                                : prm.ws + ((int64_t)(2 * (int64_t)(DYN ? share_pos(chunk, prm.nchunks)
                                                                                : blockIdx.x) +
                                                         (p == pa ? 0 : 1)) * TMV) * (128 * NT);
      const int64_t ostride = full ? N : 128 * NT;
      const uint32_t slot = pc % L::kSlots;
#if HRPB_EPI_SLEEP > 0
      if (!tracing(prm)) mbar_wait_backoff(&tfull[slot], (pc / L::kSlots) & 1, HRPB_EPI_SLEEP);
      else
#endif
      mbar_wait_acc(prm, &tfull[slot], (pc / L::kSlots) & 1, wacc);
      if (et == 0) trace_ev(prm, 5, pc);
      tc_fence_after();
      // rows per tcgen05.wait: 32 for one set; with kMW sets 16 rows of every written set are loaded before one
      // wait and summed in set order (kMW x 16 registers; 512 threads leave 128 per thread)
      constexpr int kRows = kMW > 1 ? 16 : (TMV < 32 ? TMV : 32);
      const uint32_t tq = tbase + ((uint32_t)(32 * qd) << 16) + slot * L::kSetCols;
#pragma unroll
      for (int t = 0; t < NT; ++t) {
#pragma unroll
        for (int h0 = 0; h0 < TMV; h0 += kRows) {
          uint32_t v[kMW][kRows / 16][16];  // panel rows [h0, h0 + kRows) of this lane's column, per set
#pragma unroll
          for (int w = 0; w < kMW; ++w)
            if ((cmask >> w) & 1u) {
#pragma unroll
              for (int c16 = 0; c16 < kRows / 16; ++c16)
                tmem_ld16(tq + w * L::kCols1 + t * TMV + h0 + c16 * 16, v[w][c16]);
            }
          tmem_ld_wait();
          float a[kRows];  // sum of the written sets in set order (the first one copied: -0.0 stays -0.0)
          bool first = true;
#pragma unroll
          for (int w = 0; w < kMW; ++w)
            if ((cmask >> w) & 1u) {
#pragma unroll
              for (int r = 0; r < kRows; ++r) {
                const float x = __uint_as_float(v[w][r >> 4][r & 15]);
                a[r] = first ? x : a[r] + x;
              }
              first = false;
            }
          const int64_t c = 128 * t + 32 * qd + lane;
          if (c < ncols && !(dbg(prm, 1))) {
            float* dst = obase + c + (int64_t)h0 * ostride;
            if (RMAP && full) {  // reordered rows (NEXT-4): each row to its original C row
#pragma unroll
              for (int r = 0; r < kRows; ++r)
                if (h0 + r < nrows) __stcs(prm.C + (int64_t)prm.row_map[row0 + h0 + r] * N + n0 + c, a[r]);
            } else if (nrows == TMV) {
#pragma unroll
              for (int r = 0; r < kRows; ++r) __stcs(dst + (int64_t)r * ostride, a[r]);
            } else {
#pragma unroll
              for (int r = 0; r < kRows; ++r)
                if (h0 + r < nrows) __stcs(dst + (int64_t)r * ostride, a[r]);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      ++pc;
    }
    pc_epi = pc;
  }
  base += cbE - cbB;
  if (!DYN) break;
  // dynamic S1: every role is done with this share (the epilogue has stored its last panel, so every MMA, gather
  // and decode of it completed); claim the next share in order
  tc_fence_before();
  if (tid == 0) misc[1] = atomicAdd(prm.chunk_ctr, 1u) + gridDim.x;
  __syncthreads();
  tc_fence_after();
  chunk = misc[1];
  if (chunk >= prm.nchunks) break;
  }  // shares
  if (tracing(prm) && blockIdx.x == 0 && lane == 0) {
    prm.trace[8 * kTraceN + 2 * warp] = wacc;
    prm.trace[8 * kTraceN + 2 * warp + 1] = clock64() - t_start;
  }
  tc_fence_before();
  __syncthreads();
  if (tracing(prm) && threadIdx.x == 0 && 4 * blockIdx.x + 3 < kTraceN) {  // per-CTA balance (S1 cost model)
    long long* t = prm.trace + 9 * kTraceN + 4 * blockIdx.x;
    t[0] = clock64() - t_start;
    t[1] = (long long)range[3] - (long long)range[2];
    t[2] = (long long)range[1] - (long long)range[0];
    t[3] = (long long)range[0];
  }
  if (warp == kMmaWarp) {
    tc_fence_after();
    tmem_dealloc(tbase, tmem_cols);
  }
  if (prm.cta_t && tid == 0) {
    prm.cta_t[4 * blockIdx.x + 1] = (long long)globaltimer();
    prm.cta_t[4 * blockIdx.x + 2] = (long long)range[3] - (long long)range[2];
    prm.cta_t[4 * blockIdx.x + 3] = (long long)range[1] - (long long)range[0];
  }
}

// Dynamic S1 (Scratch::nchunks > 0): the ranges of all shares, one warp each, before k_spmm (which then only
// reads them as its CTAs claim shares), and the claim counter reset.
template <uint64_t PW>
__global__ void __launch_bounds__(128) k_spmm_chunks(const uint32_t* __restrict__ brp, int64_t p_lo, int64_t p_hi,
                                                     uint32_t nchunks, uint64_t* __restrict__ ranges,
                                                     uint64_t* split_flag, uint64_t epoch, uint32_t* ctr) {
  pdl_wait();
  if (blockIdx.x == 0 && threadIdx.x == 0) *ctr = 0u;
  const uint64_t c = (uint64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (c >= nchunks) return;
  // c = position of the share in the matrix (ranges, workspace tiles and the fix-up are indexed by position); it
  // is claimed as number n - 1 - c: the matrix is walked from its end (#if HRPB_DYN_REV). Guided sizes: the first
  // half of the claims are 3 fine units of a grid of 2 n (3/4 of the work), the second half 1 unit each, so the
  // shares claimed last (which decide when the launch ends) are 3x smaller.
  const uint64_t nA = nchunks / 2, F = 3 * nA + (nchunks - nA);
  auto fine = [&](uint64_t x) { return x <= nA ? 3 * x : 3 * nA + (x - nA); };  // claims -> fine units
#if HRPB_DYN_REV
  const uint64_t f0 = F - fine(nchunks - c), f1 = F - fine(nchunks - 1 - c);
#else
  const uint64_t f0 = fine(c), f1 = fine(c + 1);
#endif
  const CtaWork cw = cta_work_span<PW>(brp, p_lo, p_hi, f0, f1, F, WarpFind<PW>());
  if ((threadIdx.x & 31) == 0) {
    if (cw.bB < cw.bE && !(cw.first_full && cw.last_full)) *split_flag = epoch;
    uint64_t* rg = ranges + 4 * c;
    rg[0] = (uint64_t)cw.pa;
    rg[1] = (uint64_t)cw.pb;
    rg[2] = (uint64_t)cw.bB | ((uint64_t)cw.bE << 32);
    rg[3] = (uint64_t)cw.first_full | ((uint64_t)cw.last_full << 1);
  }
}

// S1 fix-up. CTA c reads the S1 ranges k_spmm published: if CTA c - 1's last panel q is split (boundary c lies
// strictly inside q) and boundary c is the first one inside q (CTA c - 1 starts at or before q's start), it sums
// the partial tiles of every CTA holding blocks of q, in CTA order (deterministic), and writes q's rows of C. The
// contributing CTAs are listed once per CTA in shared memory (no per-element work search).
template <int TMV>
__global__ void __launch_bounds__(kFixThreads) k_spmm_fixup(const uint32_t* __restrict__ brp,
                                                          const uint64_t* __restrict__ ranges,
                                                          const float* __restrict__ ws, float* __restrict__ C,
                                                          int64_t M, int64_t N, int n0, int wcols,
                                                          const uint64_t* split_flag, uint64_t epoch,
                                                          const int32_t* __restrict__ row_map) {
  pdl_wait();
  constexpr int kMaxSrc = 256;
  __shared__ int s_src[kMaxSrc];  // (cc << 1) | workspace slot of each contributing share, one batch
  __shared__ int s_n;
  __shared__ uint64_t s_next;     // share to continue the contributor scan from (next batch)
  __shared__ int64_t s_q;
  const uint64_t G = gridDim.x, c = blockIdx.x;
  if (c == 0 || *split_flag != epoch) return;  // no split panel in this launch
  if (threadIdx.x == 0) {
    s_n = 0;
    s_next = G;
    const uint64_t* A = ranges + 4 * (c - 1);
    const int64_t pa = (int64_t)A[0], pb = (int64_t)A[1];
    const uint32_t bB = (uint32_t)A[2], bE = (uint32_t)(A[2] >> 32);
    const bool ff = A[3] & 1, lf = (A[3] >> 1) & 1;
    const int64_t q = pb - 1;
    s_q = q;
    if (bB < bE && !lf && (pa != q || ff)) s_next = c - 1;  // boundary c is the first one strictly inside panel q
  }
  __syncthreads();
  if (s_next >= G) return;
  const int64_t q = s_q;
  const int64_t row0 = q * TMV;
  const int nrows = (int)min((int64_t)TMV, M - row0);
  const int ncols = (int)min((int64_t)wcols, N - n0);
  const uint32_t q0 = brp[q], q1 = brp[q + 1];
  // contributors in share order, in batches of kMaxSrc (a panel may span more shares than one batch holds): the
  // first batch writes C, later ones add to it — the same order of additions as one pass (deterministic)
  for (int batch = 0;; ++batch) {
    if (threadIdx.x == 0) {
      int n = 0;
      uint64_t cc = s_next;
      for (; cc < G && n < kMaxSrc; ++cc) {
        const uint64_t* W = ranges + 4 * cc;
        const int64_t wpa = (int64_t)W[0];
        if (wpa > q) { cc = G; break; }
        const uint32_t b0 = max(q0, (uint32_t)W[2]), b1 = min(q1, (uint32_t)(W[2] >> 32));
        if (b0 >= b1) continue;  // no blocks of q in share cc
        s_src[n++] = (int)(cc << 1) | (q == wpa ? 0 : 1);
      }
      s_n = n;
      s_next = cc;
    }
    __syncthreads();
    const int n = s_n;
    for (int e = threadIdx.x; e < nrows * ncols; e += kFixThreads) {
      const int r = e / ncols, col = e - r * ncols;
      const int64_t cr = row_map ? (int64_t)row_map[row0 + r] : row0 + r;
      float acc = batch == 0 ? 0.f : C[cr * N + n0 + col];
      for (int k = 0; k < n; ++k) {
        const int src = s_src[k];
        acc += ws[((int64_t)(2 * (src >> 1) + (src & 1)) * TMV + r) * wcols + col];
      }
      C[cr * N + n0 + col] = acc;
    }
    __syncthreads();
    if (s_next >= G) break;
  }
}

template <int NT, int GM, int TMV, int TKV>
static hrpb_status_t launch_nt(const hrpb_handle* h, const CUtensorMap& tm, const float* B, int64_t ldb, float* C,
                               int64_t N, int n0, int64_t p_lo, int64_t p_hi, const Scratch& scr, cudaStream_t s) {
  using L = SmemLayout<NT, TMV, TKV>;
  // producer warp w (and decoder warp w) owns blocks i = w mod 4; with S a multiple of 4 every stage is
  // only ever filled by one warp, so a warp running ahead cannot alias an mbarrier phase.
  static_assert(kDecWarps % kProdWarps == 0, "stage ownership: decoder count must be a multiple of producers");
  auto smem_for = [](int st) {
    return (size_t)1024 /*alignment*/ + (size_t)st * L::kStage + (3 * st + 8) * 8 + 128 +
           kDecWarps * L::kNbk * 12 + 16 + kProdWarps * kPfRing * (TKV + 4) * 4;
  };
  int stages = kMaxStages - kMaxStages % kDecWarps;
  while (stages > kDecWarps && smem_for(stages) > 227 * 1024) stages -= kDecWarps;
  static const int stage_cap = [] {
    const char* e = getenv("HRPB_STAGES");  // experiments: cap the pipeline depth (multiple of 4)
    return e ? atoi(e) : 0;
  }();
  if (stage_cap >= kDecWarps && stage_cap < stages) stages = stage_cap - stage_cap % kDecWarps;
  // at least half of the SM's shared memory: one CTA per SM, so a second resident CTA can never block in
  // tcgen05.alloc on the TMEM columns the first one holds (TM = 128 at N > 128 allocates all 512)
  const size_t smem = smem_for(stages) > 116 * 1024 ? smem_for(stages) : 116 * 1024;
  if (smem > 227 * 1024) return HRPB_ERROR_NOT_SUPPORTED;  // (not reachable with the instantiated NT / TM / TK)
  // dynamic S1 instantiated for the long-launch shapes only (cp.async gather, TK = 16, TM <= 32); row-mapped C
  // (NEXT-4) for the cp.async gather with TK = 16
  constexpr bool kDynOk = GM == 1 && TKV == 16 && TMV <= 32;
  constexpr bool kRmapOk = GM == 1 && TKV == 16;
  if (h->row_map && !kRmapOk) return HRPB_ERROR_NOT_SUPPORTED;
  static std::atomic<uint64_t> attr_set{0};  // per device: an attribute applies to the current device only
  if (first_on_device(attr_set)) {
    cudaError_t e = cudaFuncSetAttribute(k_spmm<NT, GM, TMV, TKV, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e == cudaSuccess && kDynOk)
      e = cudaFuncSetAttribute(k_spmm<NT, GM, TMV, TKV, kDynOk>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024);
    if (e == cudaSuccess && kRmapOk)
      e = cudaFuncSetAttribute(k_spmm<NT, GM, TMV, TKV, false, kRmapOk>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               227 * 1024);
    if (e == cudaSuccess && kDynOk && kRmapOk)
      e = cudaFuncSetAttribute(k_spmm<NT, GM, TMV, TKV, kDynOk, kRmapOk>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) {
      attr_set = 0;
      return cuda_status(e);
    }
  }
  static const char* trace_path = kInstr ? getenv("HRPB_TRACE") : nullptr;
  long long* trace = nullptr;
  if (trace_path) {
    trace = (long long*)dalloc(kTraceSlots * kTraceN * sizeof(long long), s);
    cudaMemsetAsync(trace, 0, kTraceSlots * kTraceN * sizeof(long long), s);
  }
  static const int debug = [] {
    const char* e = kInstr ? getenv("HRPB_DEBUG") : nullptr;
    return e ? atoi(e) : 0;
  }();
  int grid = num_sms();
  if ((int64_t)grid > p_hi - p_lo) grid = (int)(p_hi > p_lo ? p_hi - p_lo : 1);
  static const char* cta_path = getenv("HRPB_CTA_TIMES");  // diagnostics: per-CTA wall times of this launch
  long long* cta_t = nullptr;
  if (cta_path) {
    cta_t = (long long*)dalloc(4 * (size_t)grid * sizeof(long long), s);
    cudaMemsetAsync(cta_t, 0, 4 * (size_t)grid * sizeof(long long), s);
  }
  SpmmParams prm{h->brp, h->ac, h->sp, h->packed, C, h->M, N, h->P, h->NB, p_lo, p_hi, scr.ws, scr.flag, scr.epoch,
                 scr.ranges, B, h->K, ldb, n0, stages, trace, {}, 0u, 0.f, 0, 0u, nullptr, h->row_map, nullptr,
                 debug};
  if (GM == 2) {
    if (!scr.sd) return HRPB_ERROR_INVALID_VALUE;
    for (int r = 0; r < scr.sd->nsh; ++r) prm.sh_ptr[r] = scr.sd->ptr[r];
    prm.sh_rps = scr.sd->rps;
    prm.sh_inv = 1.0f / (float)scr.sd->rps;
    prm.nsh = scr.sd->nsh;
  }
  prm.cta_t = cta_t;
  const uint32_t nch = kDynOk && scr.nchunks >= (uint32_t)grid ? scr.nchunks : 0u;  // dynamic S1 (shares >= CTAs)
  if (nch) {
    prm.nchunks = nch;
    prm.chunk_ctr = scr.ctr;
    launch_pdl(k_spmm_chunks<panel_weight<TMV>()>, (nch + 3) / 4, 128, 0, s, h->brp, p_lo, p_hi, nch, scr.ranges,
               scr.flag, scr.epoch, scr.ctr);
    note_launch();
  }
  const bool rmap = h->row_map != nullptr;
  if (nch && rmap) launch_pdl(k_spmm<NT, GM, TMV, TKV, kDynOk, kRmapOk>, grid, kSpmmThreads, smem, s, tm, prm);
  else if (nch) launch_pdl(k_spmm<NT, GM, TMV, TKV, kDynOk>, grid, kSpmmThreads, smem, s, tm, prm);
  else if (rmap) launch_pdl(k_spmm<NT, GM, TMV, TKV, false, kRmapOk>, grid, kSpmmThreads, smem, s, tm, prm);
  else launch_pdl(k_spmm<NT, GM, TMV, TKV, false>, grid, kSpmmThreads, smem, s, tm, prm);
  if (cta_t) {  // (blocks the stream: diagnostics only)
    std::vector<long long> host(4 * (size_t)grid);
    cudaMemcpyAsync(host.data(), cta_t, host.size() * sizeof(long long), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (FILE* f = fopen(cta_path, "wb")) {
      fwrite(host.data(), sizeof(long long), host.size(), f);
      fclose(f);
    }
    dfree(cta_t, s);
  }
  launch_pdl(k_spmm_fixup<TMV>, nch ? (int)nch : grid, kFixThreads, 0, s, h->brp, (const uint64_t*)scr.ranges, scr.ws, C,
             h->M, N, n0, 128 * NT, scr.flag, scr.epoch, h->row_map);
  note_launch(2);
  if (trace) {  // debugging aid: dump CTA 0's per-block timestamps (blocks the stream)
    static long long host[kTraceSlots * kTraceN];
    cudaMemcpyAsync(host, trace, sizeof(host), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    if (FILE* f = fopen(trace_path, "wb")) {
      fwrite(host, sizeof(host), 1, f);
      fclose(f);
    }
    dfree(trace, s);
  }
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HRPB_SUCCESS : cuda_status(e);
}

// one translation unit per TK instantiates its kernels (parallel compilation): spmm_tk16.cu, spmm_tk32.cu; the
// row-sharded B variant (GM = 2) for both TK in spmm_sharded.cu
hrpb_status_t spmm_dispatch_sharded(const hrpb_handle* h, const CUtensorMap& tm, float* C, int64_t N, int n0, int nt,
                                    int64_t p_lo, int64_t p_hi, const Scratch& scr, cudaStream_t s);
template <int TKV>
hrpb_status_t spmm_dispatch(const hrpb_handle* h, const CUtensorMap& tm, const float* Bt, int64_t ld, float* C,
                            int64_t N, int n0, int nt, int gm, int64_t p_lo, int64_t p_hi, const Scratch& scr,
                            cudaStream_t s);

}  // namespace hrpb
