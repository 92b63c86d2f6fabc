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
#include <mutex>

#include "common.cuh"
#include "internal.h"

namespace hrpb {

constexpr int kSpmmThreads = 224;  // 7 warps
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

template <int NT>
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
      mbar_init(&full_b[s], 1);
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
  if (warp == 2) tmem_alloc(&misc[0], tmem_cols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = misc[0];
  const int64_t pa = range[0], pb = range[1];
  const uint32_t* __restrict__ brp = prm.brp;
  const int n0 = prm.n0;
  const int64_t N = prm.N, M = prm.M;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      const uint64_t pol_a = policy_evict_first();
      const int na_eff = (int)min((int64_t)L::kNA, ceil_div(N - n0, 32));  // atoms with any column < N
      const uint32_t b_bytes = 16u * 128u * (uint32_t)na_eff;
      uint32_t i = 0;
      const int64_t b_begin = brp[pa], b_end = brp[pb];
      for (int64_t b = b_begin; b < b_end; ++b, ++i) {
        const int s = i % S;
        const uint32_t ph = (i / S) & 1;
        const uint4* acv = reinterpret_cast<const uint4*>(prm.ac + b * 16);
        uint4 c0 = __ldg(acv), c1 = __ldg(acv + 1), c2 = __ldg(acv + 2), c3 = __ldg(acv + 3);
        const uint64_t s0 = __ldg(prm.sp + b), s1 = __ldg(prm.sp + b + 1);
        mbar_wait(&empty[s], ph ^ 1);
        const uint32_t a_bytes = (uint32_t)(s1 - s0);
        mbar_expect_tx(&full_a[s], a_bytes);
        bulk_g2s(araw0 + (size_t)s * kARawBytes, prm.packed + s0, a_bytes, &full_a[s], pol_a);
        mbar_expect_tx(&full_b[s], b_bytes);
        uint8_t* bt = btile0 + (size_t)s * L::kBTile;
        const uint4 rows[4] = {c0, c1, c2, c3};
#pragma unroll
        for (int g4 = 0; g4 < 4; ++g4) {
          for (int a = 0; a < na_eff; ++a) {
            tma_gather4(bt + (g4 * L::kNA + a) * 512, &tmB, n0 + 32 * a, (int32_t)rows[g4].x, (int32_t)rows[g4].y,
                        (int32_t)rows[g4].z, (int32_t)rows[g4].w, &full_b[s]);
          }
        }
      }
    }
  } else if (warp == 1) {
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
  } else if (warp == 2) {
    // ---------------------------------------------------------------- MMA issuer (one thread)
    if (lane == 0) {
      uint32_t i = 0, pc = 0;
      const uint32_t bt0 = smem_u32(btile0), at0 = smem_u32(atile0);
      for (int64_t p = pa; p < pb; ++p) {
        const int64_t bb = brp[p], be = brp[p + 1];
        if (bb == be) continue;
        const uint32_t slot = pc & 1;
        mbar_wait(&tempty[slot], ((pc >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dcol = tbase + slot * NT * 16;
        for (int64_t b = bb; b < be; ++b, ++i) {
          const int s = i % S;
          const uint32_t ph = (i / S) & 1;
          mbar_wait(&full_b[s], ph);
          mbar_wait(&dec[s], ph);
          tc_fence_after();
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
        umma_commit(&tfull[slot]);
        ++pc;
      }
    }
    __syncwarp();
  } else {
    // ---------------------------------------------------------------- epilogue (warps 3..6)
    const int qd = warp & 3;            // TMEM lane quadrant accessible to this warp
    const int et = tid - 96;            // 0..127
    const int64_t ncols = min((int64_t)128 * NT, N - n0);
    uint32_t pc = 0;
    for (int64_t p = pa; p < pb; ++p) {
      const int64_t row0 = p * 16;
      const int nrows = (int)min((int64_t)16, M - row0);
      if (brp[p] == brp[p + 1]) {  // empty panel: zero rows (R13)
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
  if (warp == 2) {
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

template <int NT>
static hrpb_status_t launch_nt(const hrpb_handle* h, const CUtensorMap& tm, float* C, int64_t N, int n0,
                               cudaStream_t s) {
  using L = SmemLayout<NT>;
  const int budget = 227 * 1024 - 1024 /*alignment*/ - 512 /*barriers, misc*/;
  int stages = budget / L::kStage;
  if (stages > kMaxStages) stages = kMaxStages;
  const size_t smem = 1024 + (size_t)stages * L::kStage + (4 * stages + 4) * 8 + 64;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(k_spmm<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    if (e != cudaSuccess) return cuda_status(e);
    attr_set = true;
  }
  SpmmParams prm{h->brp, h->ac, h->sp, h->packed, C, h->M, N, h->P, h->NB, n0, stages};
  int grid = num_sms();
  if ((int64_t)grid > h->P) grid = (int)(h->P > 0 ? h->P : 1);
  k_spmm<NT><<<grid, kSpmmThreads, smem, s>>>(tm, prm);
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
    switch (nt) {
      case 1: st = launch_nt<1>(h, tm, C, N, (int)n0, s); break;
      case 2: st = launch_nt<2>(h, tm, C, N, (int)n0, s); break;
      case 3: st = launch_nt<3>(h, tm, C, N, (int)n0, s); break;
      default: st = launch_nt<4>(h, tm, C, N, (int)n0, s); break;
    }
    if (st != HRPB_SUCCESS) return st;
  }
  return HRPB_SUCCESS;
}

}  // namespace hrpb
