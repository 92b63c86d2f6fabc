// spmm.cu — host side of hrpb_spmm_sm100: B row-pitch padding, the B tensor map, N-tile loop and the panel-range
// entry points, and the row-sharded B entry point (NEXT-3) (the kernel itself is in spmm_kernel.cuh, instantiated per TK
// in spmm_tk16.cu / spmm_tk32.cu, the row-sharded variant in spmm_sharded.cu).
#include <cstring>

#include "spmm_kernel.cuh"

namespace hrpb {

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

hrpb_status_t spmm_impl(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, cudaStream_t s) {
  return spmm_range_impl(h, B, ldb, C, N, 0, h->P, s);
}

hrpb_status_t spmm_range_impl(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, int64_t p_lo,
                              int64_t p_hi, cudaStream_t s) {
  return spmm_core(h, B, ldb, C, N, p_lo, p_hi, nullptr, s);
}

// NEXT-3: B row-sharded over devices (shard r = rows [r rps, min((r + 1) rps, K)), ld = N). No padded copy: every
// shard must be 16-B aligned with N % 4 == 0, and the gather runs as cp.async (GM = 2).
hrpb_status_t spmm_sharded_impl(const hrpb_handle* h, const float* const* shards, int32_t nshards,
                                int64_t rows_per_shard, float* C, int64_t N, cudaStream_t s) {
  if (nshards < 1 || nshards > kMaxShards || rows_per_shard < 1 || rows_per_shard >= (1ll << 31))
    return HRPB_ERROR_INVALID_VALUE;
  if (ceil_div(h->K, rows_per_shard) != nshards && !(h->K == 0 && nshards == 1)) return HRPB_ERROR_INVALID_VALUE;
  if (N % 4) return HRPB_ERROR_INVALID_VALUE;
  ShardDesc sd{};
  int dev = 0;
  cudaGetDevice(&dev);
  for (int r = 0; r < nshards; ++r) {
    if (!shards[r] || (reinterpret_cast<uintptr_t>(shards[r]) & 15)) return HRPB_ERROR_INVALID_VALUE;
    sd.ptr[r] = shards[r];
    // a shard in another GPU's memory (CUDA IPC mapping): enable peer access from this device once per pair
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, shards[r]) == cudaSuccess && at.type == cudaMemoryTypeDevice &&
        at.device != dev && dev >= 0 && dev < 64 && at.device >= 0 && at.device < 64) {
      static std::atomic<uint64_t> enabled[64];
      if (!(enabled[dev].load() >> at.device & 1)) {
        const cudaError_t e = cudaDeviceEnablePeerAccess(at.device, 0);
        if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) return cuda_status(e);
        cudaGetLastError();  // (clears cudaErrorPeerAccessAlreadyEnabled)
        enabled[dev].fetch_or(1ull << at.device);
      }
    }
  }
  sd.rps = (uint32_t)rows_per_shard;
  sd.nsh = nshards;
  return spmm_core(h, shards[0], N, C, N, 0, h->P, &sd, s);
}

hrpb_status_t spmm_core(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, int64_t p_lo,
                        int64_t p_hi, const ShardDesc* sd, cudaStream_t s) {
  if (N == 0 || h->M == 0 || p_hi <= p_lo) return HRPB_SUCCESS;
  if (h->NB == 0 && !h->row_map) {  // A has no entries: C = 0 (rows of the range; NB < 0 = not known yet: the kernel
    // copes; so does it with a row map, whose rows are not contiguous)
    const int64_t r0 = p_lo * h->tm, r1 = p_hi * h->tm < h->M ? p_hi * h->tm : h->M;
    cudaError_t e = cudaMemsetAsync(C + r0 * N, 0, (size_t)(r1 - r0) * N * sizeof(float), s);
    return e == cudaSuccess ? HRPB_SUCCESS : cuda_status(e);
  }
  if (!tile_supported(h->tm, h->tk)) return HRPB_ERROR_NOT_SUPPORTED;
  if (const char* pm = getenv("HRPB_L2_PERSIST_MB")) {  // experiment: L2 set-aside for evict_last lines
    static std::once_flag once;
    std::call_once(once, [pm] { cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)atoll(pm) << 20); });
  }
  EncodeTiledFn enc = get_encode();
  if (!enc) return HRPB_ERROR_NOT_SUPPORTED;
  // per-call scratch, stream-ordered on s (a handle may serve concurrent calls on different streams): the padded
  // B copy when its rows are not 16-B aligned, and the split-panel workspace of the S1 fix-up
  const float* Bt = B;
  int64_t ld = ldb;
  float* bpad = nullptr;
  if (!sd && ((reinterpret_cast<uintptr_t>(B) & 15) || (ld * 4) % 16)) {
    const int64_t ldp = align_up(N, 4);
    bpad = (float*)dalloc((size_t)h->K * ldp * sizeof(float), s);
    if (!bpad) return HRPB_ERROR_OUT_OF_MEMORY;
    k_pad_rows<<<4 * num_sms(), 256, 0, s>>>(B, h->K, N, ldb, bpad, ldp);
    note_launch();
    Bt = bpad;
    ld = ldp;
  }
  // S1 shares: one per CTA (static), or kDynShares per SM claimed dynamically on long launches (DESIGN.md §6 S1:
  // the static cost model leaves c3's CTAs at 1.15x max/mean; the share claimed last ends at most about one share
  // after the mean). The host cannot see the block count of an asynchronous build, so "long" is read from nnz.
  const int64_t ncols_max = N < 512 ? N : 512;
  // (HRPB_STATIC_S1 / HRPB_DYN_S1: force either, for experiments and the parity tests of small matrices)
  const int64_t shares = min((int64_t)kDynShares * num_sms(), p_hi - p_lo);
  // (whole-matrix launches only: the chunked launches of the pipelined host path are short)
  const bool dyn = getenv("HRPB_STATIC_S1") == nullptr && h->tm <= 32 && shares >= num_sms() &&
                   ((h->nnz >= kDynMinNnz && p_lo == 0 && p_hi == h->P) || getenv("HRPB_DYN_S1") != nullptr);
  const uint32_t nchunks = dyn ? (uint32_t)shares : 0u;
  // shares x 2 tiles x TM x (128 NT) partial tiles (static: TM * 128 NT <= 64 * 512 for every instantiated pair),
  // the split flag, the claim counter and the shares' S1 ranges
  const size_t ws_bytes = dyn ? (size_t)nchunks * 2 * h->tm * (size_t)(ceil_div(ncols_max, 128) * 128) * sizeof(float)
                              : (size_t)num_sms() * 2 * 64 * 512 * sizeof(float);
  const size_t nshares = dyn ? nchunks : (size_t)num_sms();
  float* ws = (float*)dalloc(ws_bytes + 64 + nshares * 4 * sizeof(uint64_t), s);
  if (!ws) {
    dfree(bpad, s);
    return HRPB_ERROR_OUT_OF_MEMORY;
  }
  uint64_t* flag = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(ws) + ws_bytes);
  Scratch scr{ws, flag, next_epoch(), flag + 8, sd, nchunks, reinterpret_cast<uint32_t*>(flag + 4)};
  CUtensorMap tm;
  memset(&tm, 0, sizeof(tm));  // (unused by the row-sharded cp.async gather: passed zeroed)
  if (!sd) {
    cuuint64_t gdim[2] = {(cuuint64_t)N, (cuuint64_t)h->K};
    cuuint64_t gstr[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {32, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(Bt), gdim, gstr, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      dfree(ws, s);
      dfree(bpad, s);
      return HRPB_ERROR_INVALID_VALUE;
    }
  }
  // columns per launch: NT <= 4, or <= 2 at TK = 32 (twice the stage size) and TM = 128 (two TMEM slots of
  // 2 x 128 columns fill the 512 TMEM columns)
  int64_t ncols = (h->tk == 32 || h->tm == 128) ? 256 : 512;
  if (const char* nc = getenv("HRPB_NCOLS")) {  // experiment: columns per launch (multiple of 128)
    const int64_t v = atoll(nc);
    if (v >= 128 && v % 128 == 0 && v < ncols) ncols = v;
  }
  for (int64_t n0 = 0; n0 < N; n0 += ncols) {
    const int64_t w = N - n0 < ncols ? N - n0 : ncols;
    const int nt = (int)ceil_div(w, 128);
    hrpb_status_t st;
    // B-row staging (S3): 1 = cp.async 16-B copies (default), 0 = TMA tile::gather4 (TK = 16 only; slower on
    // every config measured, kept selectable per call and parity-tested)
    const char* genv = getenv("HRPB_GATHER");
    const int gm = genv ? atoi(genv) : 1;
    if (sd) st = spmm_dispatch_sharded(h, tm, C, N, (int)n0, nt, p_lo, p_hi, scr, s);
    else if (h->tk == 16) st = spmm_dispatch<16>(h, tm, Bt, ld, C, N, (int)n0, nt, gm, p_lo, p_hi, scr, s);
    else st = spmm_dispatch<32>(h, tm, Bt, ld, C, N, (int)n0, nt, 1, p_lo, p_hi, scr, s);
    if (st != HRPB_SUCCESS) {
      dfree(ws, s);
      dfree(bpad, s);
      return st;
    }
  }
  dfree(ws, s);
  dfree(bpad, s);
  return HRPB_SUCCESS;
}

// Largest real active column of every panel of each chunk (chunk c = panels [c * per, (c + 1) * per)); the
// pipelined host entry point starts a chunk's SpMM once B rows up to that column have arrived.
__global__ void k_chunk_maxcol(const uint32_t* __restrict__ brp, const uint32_t* __restrict__ ac, int64_t P, int tk,
                               uint32_t K, int64_t per, int* __restrict__ out) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b0 = brp[p], b1 = brp[p + 1];
    if (b1 == b0) continue;
    int mx = -1;
    for (int64_t t = b1 * tk - 1; t >= b0 * tk && t >= b1 * tk - tk; --t) {  // sentinels only in the last block
      const uint32_t c = ac[t];
      if (c < K) { mx = (int)c; break; }
    }
    if (mx >= 0) atomicMax(&out[p / per], mx);
  }
}

hrpb_status_t chunk_maxcol(const hrpb_handle* h, int64_t per, int nchunks, int* dev_out, cudaStream_t s) {
  cudaError_t e = cudaMemsetAsync(dev_out, 0xFF, nchunks * sizeof(int), s);  // -1: chunk needs no B row
  if (e != cudaSuccess) return cuda_status(e);
  if (h->P > 0 && h->NB > 0) {
    k_chunk_maxcol<<<(unsigned)ceil_div(h->P, 256) < 4096 ? (unsigned)ceil_div(h->P, 256) : 4096u, 256, 0, s>>>(
        h->brp, h->ac, h->P, h->tk, (uint32_t)h->K, per, dev_out);
    note_launch();
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? HRPB_SUCCESS : cuda_status(e);
}

}  // namespace hrpb
