// spmm.cu — hrpb_spmm_sm100: C = A.B with A in HRPB.
//
// Paper kernel (Alg. "cuTeSpMM kernel design"; prose P:L244-282): one thread block
// per row panel, warps along N, SM_A/SM_B staging, per-brick pattern decode with prefix popcounts
// (P:L207-219), Ampere mma.sync m16n8k4 TF32 accumulating in registers.
//
// B200 design:
//  * persistent CTAs (one per SM), each owning a contiguous panel range balanced on
//    (blocks + panels) (S1);
//  * warp 0: TMA producer — cp.async.bulk of the packed block bytes (S2) and
//    cp.async.bulk.tensor.2d.tile::gather4 of the 16 B rows named by activeCols into an
//    MN-major SWIZZLE_128B_BASE32B tile (S3); sentinel column K is out of bounds -> zero fill;
//  * warp 1: decoder — lane l expands bits l and l+32 of every brick (prefix popcounts)
//    into a zero-filled K-major TF32 tile (cvt.rna on A, reading R15) (S2);
//  * warp 2: one thread issues tcgen05.mma.kind::tf32 computing the transposed product
//    D[n, r] += sum_k Bg[k, n] * A[r, k]  (M = 128 dense columns, N = TM = 16 panel rows, K = 8 x 2),
//    accumulating a whole panel in TMEM (double-buffered across panels) (S4);
//  * warps 3..6: epilogue — tcgen05.ld 32x32b, coalesced 128-B row stores of C (S5);
//  * mbarrier rings: full_a/full_b (TMA), dec (decoder), empty (tcgen05.commit), tfull/tempty.
#include <cstdio>
#include <cstdlib>
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace hrpb {

constexpr int kSpmmThreads = 320;  // 10 warps: 4 producers, decoder, MMA, 4 epilogue
constexpr int kProdWarps = 4;
constexpr int kARawBytes = 1152;   // >= 1072 (largest TM=16/TK=16 block), multiple of 128
constexpr int kATileBytes = 1024;  // 16 x 16 fp32 decoded block
constexpr int kMaxStages = 16;

struct SpmmParams {
  const uint32_t* brp;
  const uint32_t* ac;
  const uint64_t* sp;
  const uint8_t* packed;
  float* C;
  int64_t M, N, P, NB;
  const float* B;  // row-major K x ldb (cp.async gather mode)
  int64_t K, ldb;
  int n0;      // first output column of this launch
  int stages;  // pipeline depth
};

// instruction descriptor: D F32, A/B TF32, A MN-major, B K-major, N = 16, M = 128
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (0u << 16) | ((16u >> 3) << 17) |
                            ((128u >> 4) << 24);

template <int NT>
struct SmemLayout {
  static constexpr int kNA = 4 * NT;                 // 32-column atoms per 4-row group
  static constexpr int kBTile = 16 * 128 * 4 * NT;  // gathered rows per stage
  static constexpr int kStage = kBTile + kARawBytes + kATileBytes;
};

__device__ __forceinline__ int64_t panel_lower_bound(const uint32_t* brp, int64_t P, uint64_t target) {
  // first p in [0, P] with brp[p] + p >= target (brp[p] + p strictly increasing)
  int64_t lo = 0, hi = P;
  while (lo < hi) {
    int64_t mid = (lo + hi) >> 1;
    if ((uint64_t)brp[mid] + (uint64_t)mid >= target) hi = mid;
    else lo = mid + 1;
  }
  return lo;
}

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
__device__ __forceinline__ void cp_async_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// GM = gather mode: 0 = TMA tile::gather4 (one issuing lane per producer warp),
//                   1 = cp.async 16-B copies by all 128 producer threads into the same swizzled layout.
template <int NT, int GM>
__global__ void __launch_bounds__(kSpmmThreads, 1) k_spmm(const __grid_constant__ CUtensorMap tmB, SpmmParams prm) {
  using L = SmemLayout<NT>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  const int S = prm.stages;
  uint8_t* btile0 = smem;                                 // S x kBTile (1024-aligned)
  uint8_t* araw0 = smem + (size_t)S * L::kBTile;          // S x kARawBytes
  uint8_t* atile0 = araw0 + (size_t)S * kARawBytes;       // S x kATileBytes
  uint64_t* bars = (uint64_t*)(atile0 + (size_t)S * kATileBytes);
  uint64_t* full_a = bars;
  uint64_t* full_b = bars + S;
  uint64_t* dec = bars + 2 * S;
  uint64_t* empty = bars + 3 * S;
  uint64_t* tfull = bars + 4 * S;
  uint64_t* tempty = tfull + 2;
  uint32_t* misc = (uint32_t*)(tempty + 2);  // [0] tmem base, [2..3] panel range
  int64_t* range = (int64_t*)(misc + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t tmem_cols = NT == 1 ? 32 : (NT == 2 ? 64 : 128);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full_a[s], 1);
      mbar_init(&full_b[s], GM == 0 ? kProdWarps : kProdWarps * 32);
      mbar_init(&dec[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 4); }
    fence_mbar_init();
    // S1: contiguous panel range with ~equal (blocks + panels)
    const uint64_t W = (uint64_t)prm.NB + (uint64_t)prm.P;
    const uint64_t G = gridDim.x, c = blockIdx.x;
    range[0] = panel_lower_bound(prm.brp, prm.P, c * W / G);
    range[1] = c + 1 == G ? prm.P : panel_lower_bound(prm.brp, prm.P, (c + 1) * W / G);
    prefetch_tmap(&tmB);
  }
  if (warp == 5) tmem_alloc(&misc[0], tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = misc[0];
  const int64_t pa = range[0], pb = range[1];
  const uint32_t* __restrict__ brp = prm.brp;
  const int n0 = prm.n0;
  const int64_t N = prm.N, M = prm.M;

  if (warp < kProdWarps) {
    // ---------------------------------------------------------------- producers (warps 0..3)
    // Warp w stages rows 4w..4w+3 of every block's gathered B tile (S3); warp 0 also copies the
    // packed block bytes (S2). Metadata of 32 consecutive blocks is fetched by one coalesced load per
    // warp (lane l: block base + l), one chunk ahead, so no global latency sits between two issues.
    const uint64_t pol_a = policy_evict_first();
    const int na_eff = (int)min((int64_t)L::kNA, ceil_div(N - n0, 32));  // 32-col atoms with a column < N
    const int64_t b_begin = brp[pa], b_end = brp[pb];
    const int pw = warp;
    uint4 cur = make_uint4(0, 0, 0, 0), nxt = make_uint4(0, 0, 0, 0);
    uint64_t cs0 = 0, cs1 = 0, ns0 = 0, ns1 = 0;
    auto load_chunk = [&](int64_t base, uint4& r, uint64_t& s0, uint64_t& s1) {
      const int64_t bl = base + lane;
      if (bl < b_end) {
        r = __ldg(reinterpret_cast<const uint4*>(prm.ac + bl * 16) + pw);
        if (pw == 0) {
          s0 = __ldg(prm.sp + bl);
          s1 = __ldg(prm.sp + bl + 1);
        }
      }
    };
    if (b_begin < b_end) load_chunk(b_begin, cur, cs0, cs1);
    const uint32_t bt0 = smem_u32(btile0);
    uint32_t i = 0;
    for (int64_t base = b_begin; base < b_end; base += 32) {
      if (base + 32 < b_end) load_chunk(base + 32, nxt, ns0, ns1);
      const int cnt = (int)min((int64_t)32, b_end - base);
      for (int j = 0; j < cnt; ++j, ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        const uint32_t r0 = __shfl_sync(0xffffffffu, cur.x, j), r1 = __shfl_sync(0xffffffffu, cur.y, j);
        const uint32_t r2 = __shfl_sync(0xffffffffu, cur.z, j), r3 = __shfl_sync(0xffffffffu, cur.w, j);
        uint64_t s0 = 0, s1 = 0;
        if (pw == 0) { s0 = __shfl_sync(0xffffffffu, cs0, j); s1 = __shfl_sync(0xffffffffu, cs1, j); }
        mbar_wait(&empty[s], ph ^ 1);
        if (pw == 0 && lane == 0) {
          const uint32_t a_bytes = (uint32_t)(s1 - s0);
          mbar_expect_tx(&full_a[s], a_bytes);
          bulk_g2s(araw0 + (size_t)s * kARawBytes, prm.packed + s0, a_bytes, &full_a[s], pol_a);
        }
        const uint32_t bt = bt0 + s * L::kBTile + pw * L::kNA * 512;  // this warp's 4-row group
        if constexpr (GM == 0) {
          if (lane == 0) {
            mbar_expect_tx(&full_b[s], 4u * 128u * (uint32_t)na_eff);
            uint8_t* btg = btile0 + (size_t)s * L::kBTile + pw * L::kNA * 512;
            for (int a = 0; a < na_eff; ++a)
              tma_gather4(btg + a * 512, &tmB, n0 + 32 * a, (int32_t)r0, (int32_t)r1, (int32_t)r2, (int32_t)r3,
                          &full_b[s]);
          }
        } else {
          // lane copies 16-B chunk c = lane + 32 t of each of the 4 rows; destination follows the UMMA
          // SWIZZLE_128B_BASE32B MN-major atom (4 rows x 128 B, 32-B granule g stored at g ^ row)
          const uint32_t rows[4] = {r0, r1, r2, r3};
#pragma unroll
          for (int rr = 0; rr < 4; ++rr) {
            const bool real = rows[rr] < (uint32_t)prm.K;  // sentinel K -> zero fill
            const float* src_row = prm.B + (int64_t)(real ? rows[rr] : 0) * prm.ldb + n0;
#pragma unroll
            for (int t = 0; t < NT; ++t) {
              const int c = lane + 32 * t;  // 16-B chunk along N
              const int a = c >> 3;         // atom
              if (a < na_eff) {
                const int g = (c >> 1) & 3, h = c & 1;
                const uint32_t dst = bt + a * 512 + rr * 128 + ((g ^ rr) << 5) + (h << 4);
                const bool inb = real && (n0 + 4 * c) < N;
                cp_async16(dst, src_row + 4 * c, inb ? 16u : 0u);
              }
            }
          }
          cp_async_arrive_noinc(&full_b[s]);
        }
        __syncwarp();
      }
      cur = nxt;
      cs0 = ns0;
      cs1 = ns1;
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------------- decoder
    uint32_t i = 0;
    const int64_t b_begin = brp[pa], b_end = brp[pb];
    for (int64_t b = b_begin; b < b_end; ++b, ++i) {
      const int s = i % S;
      const uint32_t ph = (i / S) & 1;
      mbar_wait(&full_a[s], ph);
      const uint8_t* blk = araw0 + (size_t)s * kARawBytes;
      float* tile = reinterpret_cast<float*>(atile0 + (size_t)s * kATileBytes);
      const uint32_t cp = *reinterpret_cast<const uint32_t*>(blk);  // colPtr[0..3]
      const uint32_t nbr = blk[4];
      const uint32_t hdr = (5 + nbr + 7) & ~7u;
      const uint64_t* pats = reinterpret_cast<const uint64_t*>(blk + hdr);
      const float* vals = reinterpret_cast<const float*>(blk + hdr + 8 * nbr);
      const uint32_t below = (1u << lane) - 1u;
      uint32_t off = 0;
#pragma unroll
      for (int bc = 0; bc < 4; ++bc) {
        const uint32_t k0 = (cp >> (8 * bc)) & 0xFF;
        const uint32_t k1 = bc < 3 ? (cp >> (8 * (bc + 1))) & 0xFF : nbr;
        float v0 = 0.f, v1 = 0.f;
        if (k1 > k0) {  // TM = 16: at most one brick per brick column
          const uint64_t pt = pats[k0];
          const uint32_t lo = (uint32_t)pt, hi = (uint32_t)(pt >> 32);
          if ((lo >> lane) & 1u) v0 = vals[off + __popc(lo & below)];
          if ((hi >> lane) & 1u) v1 = vals[off + __popc(lo) + __popc(hi & below)];
          off += __popc(lo) + __popc(hi);
        }
        tile[bc * 64 + lane] = to_tf32_rna(v0);
        tile[bc * 64 + 32 + lane] = to_tf32_rna(v1);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dec[s]);
    }
  } else if (warp == 5) {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    uint32_t i = 0, pc = 0;
    const uint32_t bt0 = smem_u32(btile0), at0 = smem_u32(atile0);
    PanelCursor cursor(brp, pa, pb, lane);
    int64_t p;
    uint32_t bb, be;
    while (cursor.next(p, bb, be)) {
      if (bb == be) continue;
      const uint32_t slot = pc & 1;
      mbar_wait(&tempty[slot], ((pc >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dcol = tbase + slot * NT * 16;
      for (uint32_t b = bb; b < be; ++b, ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        mbar_wait(&full_b[s], ph);
        mbar_wait(&dec[s], ph);
        tc_fence_after();
        if (lane == 0) {
          const uint32_t bt = bt0 + s * L::kBTile, at = at0 + s * kATileBytes;
#pragma unroll
          for (int t = 0; t < NT; ++t) {
#pragma unroll
            for (int g = 0; g < 2; ++g) {
              const uint64_t ad = umma_sdesc(bt + (2 * g * L::kNA + 4 * t) * 512, 512, L::kNA * 512, 1);
              const uint64_t bd = umma_sdesc(at + g * 512, 256, 128, 0);
              umma_tf32(dcol + t * 16, ad, bd, kIdesc, (b > bb || g > 0) ? 1u : 0u);
            }
          }
          umma_commit(&empty[s]);
        }
        __syncwarp();
      }
      if (lane == 0) umma_commit(&tfull[slot]);
      __syncwarp();
      ++pc;
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 6..9)
    const int qd = warp & 3;            // TMEM lane quadrant accessible to this warp
    const int et = tid - 192;           // 0..127
    const int64_t ncols = min((int64_t)128 * NT, N - n0);
    uint32_t pc = 0;
    PanelCursor cursor(brp, pa, pb, lane);
    int64_t p;
    uint32_t bb, be;
    while (cursor.next(p, bb, be)) {
      const int64_t row0 = p * 16;
      const int nrows = (int)min((int64_t)16, M - row0);
      if (bb == be) {  // empty panel: zero rows (R13)
        for (int r = 0; r < nrows; ++r)
          for (int64_t c = et; c < ncols; c += 128) prm.C[(row0 + r) * N + n0 + c] = 0.f;
        continue;
      }
      const uint32_t slot = pc & 1;
      mbar_wait(&tfull[slot], (pc >> 1) & 1);
      tc_fence_after();
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        uint32_t v[16];
        tmem_ld16(tbase + ((uint32_t)(32 * qd) << 16) + slot * NT * 16 + t * 16, v);
        tmem_ld_wait();
        const int64_t c = 128 * t + 32 * qd + lane;
        if (c < ncols) {
          float* dst = prm.C + row0 * N + n0 + c;
#pragma unroll
          for (int r = 0; r < 16; ++r)
            if (r < nrows) __stcs(dst + (int64_t)r * N, __uint_as_float(v[r]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[slot]);
      ++pc;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 5) {
    tc_fence_after();
    tmem_dealloc(tbase, tmem_cols);
  }
}

// pads B to a 16-byte row pitch (TMA global strides must be multiples of 16 B)
__global__ void k_pad_rows(const float* __restrict__ src, int64_t rows, int64_t n, int64_t ld, float* __restrict__ dst,
                           int64_t ldp) {
  int64_t total = rows * ldp;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = i / ldp, c = i % ldp;
    dst[i] = c < n ? src[r * ld + c] : 0.f;
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)p;
  });
  return fn;
}

template <int NT, int GM>
static hrpb_status_t launch_nt(const hrpb_handle* h, const CUtensorMap& tm, const float* B, int64_t ldb, float* C,
                               int64_t N, int n0, cudaStream_t s) {
  using L = SmemLayout<NT>;
  const int budget = 227 * 1024 - 1024 /*alignment*/ - 512 /*barriers, misc*/;
  int stages = budget / L::kStage;
  if (stages > kMaxStages) stages = kMaxStages;
  const size_t smem = 1024 + (size_t)stages * L::kStage + (4 * stages + 4) * 8 + 64;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_spmm<NT, GM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return cuda_status(e);
    attr_set = true;
  }
  SpmmParams prm{h->brp, h->ac, h->sp, h->packed, C, h->M, N, h->P, h->NB, B, h->K, ldb, n0, stages};
  int grid = num_sms();
  if ((int64_t)grid > h->P) grid = (int)(h->P > 0 ? h->P : 1);
  k_spmm<NT, GM><<<grid, kSpmmThreads, smem, s>>>(tm, prm);
  note_launch();
  cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HRPB_SUCCESS : cuda_status(e);
}

hrpb_status_t spmm_impl(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, cudaStream_t s) {
  if (N == 0 || h->M == 0) return HRPB_SUCCESS;
  if (h->NB == 0) {  // A has no entries: C = 0
    cudaError_t e = cudaMemsetAsync(C, 0, (size_t)h->M * N * sizeof(float), s);
    return e == cudaSuccess ? HRPB_SUCCESS : cuda_status(e);
  }
  if (h->tm != 16 || h->tk != 16) return HRPB_ERROR_NOT_SUPPORTED;
  EncodeTiledFn enc = get_encode();
  if (!enc) return HRPB_ERROR_NOT_SUPPORTED;
  const float* Bt = B;
  int64_t ld = ldb;
  if ((reinterpret_cast<uintptr_t>(B) & 15) || (ld * 4) % 16) {
    const int64_t ldp = align_up(N, 4);
    const size_t need = (size_t)h->K * ldp * sizeof(float);
    hrpb_handle* hm = const_cast<hrpb_handle*>(h);
    if (hm->bpad_bytes < need) {
      if (hm->bpad) dfree(hm->bpad, s);
      hm->bpad = (float*)dalloc(need, s);
      hm->bpad_bytes = hm->bpad ? need : 0;
      if (!hm->bpad) return HRPB_ERROR_OUT_OF_MEMORY;
    }
    k_pad_rows<<<4 * num_sms(), 256, 0, s>>>(B, h->K, N, ldb, hm->bpad, ldp);
    note_launch();
    Bt = hm->bpad;
    ld = ldp;
  }
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)h->K};
  cuuint64_t gstr[1] = {(cuuint64_t)ld * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(Bt), gdim, gstr, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return HRPB_ERROR_INVALID_VALUE;
  for (int64_t n0 = 0; n0 < N; n0 += 512) {
    const int64_t w = N - n0 < 512 ? N - n0 : 512;
    const int nt = (int)ceil_div(w, 128);
    hrpb_status_t st;
    static const int gm = [] {
      const char* e = getenv("HRPB_GATHER");  // 0 = TMA gather4, 1 = cp.async (default)
      return e ? atoi(e) : 1;
    }();
    if (gm == 0) {
      switch (nt) {
        case 1: st = launch_nt<1, 0>(h, tm, Bt, ld, C, N, (int)n0, s); break;
        case 2: st = launch_nt<2, 0>(h, tm, Bt, ld, C, N, (int)n0, s); break;
        case 3: st = launch_nt<3, 0>(h, tm, Bt, ld, C, N, (int)n0, s); break;
        default: st = launch_nt<4, 0>(h, tm, Bt, ld, C, N, (int)n0, s); break;
      }
    } else {
      switch (nt) {
        case 1: st = launch_nt<1, 1>(h, tm, Bt, ld, C, N, (int)n0, s); break;
        case 2: st = launch_nt<2, 1>(h, tm, Bt, ld, C, N, (int)n0, s); break;
        case 3: st = launch_nt<3, 1>(h, tm, Bt, ld, C, N, (int)n0, s); break;
        default: st = launch_nt<4, 1>(h, tm, Bt, ld, C, N, (int)n0, s); break;
      }
    }
    if (st != HRPB_SUCCESS) return st;
  }
  return HRPB_SUCCESS;
}

}  // namespace hrpb
