// internal.h — library-internal declarations shared by api.cu, build.cu and spmm.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "../../include/hrpb.h"

struct hrpb_handle {
  int64_t M, K, nnz, P, NB, bytes;
  int32_t tm, tk;
  uint32_t* brp;    // [P+1]
  uint32_t* ac;     // [NB_cap * tk]
  uint64_t* sp;     // [NB_cap + 1]
  uint8_t* packed;  // [bytes_cap]
  cudaStream_t stream;  // build stream (frees are ordered on it)
  // streams other than `stream` that ran hrpb_spmm on this handle, with an event recorded after their latest
  // use: hrpb_free makes the build stream wait on them before the stream-ordered frees (kMaxUse distinct streams;
  // beyond that hrpb_free synchronizes the device)
  static constexpr int kMaxUse = 8;
  int n_use;
  bool use_overflow;
  cudaStream_t use_st[kMaxUse];
  cudaEvent_t use_ev[kMaxUse];
  // NEXT-4: the handle was built from a row-permuted CSR (hrpb_reorder_rows); the SpMM writes its row i to C row
  // row_map[i] (caller-owned device int32 [M]), so C = A.B in the original row order. NULL = identity.
  const int32_t* row_map;
};

namespace hrpb {

// device allocation helpers (stream-ordered pool); return nullptr on failure
void* dalloc(size_t bytes, cudaStream_t s);
void dfree(void* p, cudaStream_t s);
void note_launch(int n = 1);
hrpb_status_t cuda_status(cudaError_t e);

// deferred_info == NULL: synchronous (one stream sync, sizes and status read back). Otherwise the read-back is
// enqueued into that pinned 3-word buffer and the caller synchronizes the stream and calls build_finish.
hrpb_status_t build_impl(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                         const float* values, int32_t tm, int32_t tk, cudaStream_t s, hrpb_handle* h,
                         uint64_t* deferred_info = nullptr, bool sticky = false);
hrpb_status_t build_finish(hrpb_handle* h, const uint64_t* info, hrpb_status_t st);
// automatic TM (cfg->tm == 0): one sampling kernel over the CSR + a stream sync; *tm_out in {16, 64}; stats (if
// not NULL) = {sampled blocks at TM = 16, at TM = 64, sampled 16-row panels}
hrpb_status_t choose_tm(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                        cudaStream_t s, int32_t* tm_out, uint64_t* stats);
// synchronizes s, returns INVALID_CSR if any sticky build (sticky = true above) flagged its input since the
// last call, and clears the flag
hrpb_status_t sticky_take(cudaStream_t s);

hrpb_status_t spmm_impl(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, cudaStream_t s);
struct ShardDesc;
// common body of the SpMM entry points: panels [p_lo, p_hi); sd = NULL, or the row-sharded B of hrpb_spmm_sharded
hrpb_status_t spmm_core(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, int64_t p_lo,
                        int64_t p_hi, const ShardDesc* sd, cudaStream_t s);
// NEXT-3: B rows [r rps, min((r + 1) rps, K)) at shards[r] (ld = N), r < nshards = ceil(K / rps)
hrpb_status_t spmm_sharded_impl(const hrpb_handle* h, const float* const* shards, int32_t nshards,
                                int64_t rows_per_shard, float* C, int64_t N, cudaStream_t s);
// C rows of panels [p_lo, p_hi) only (the pipelined host entry point)
hrpb_status_t spmm_range_impl(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, int64_t p_lo,
                              int64_t p_hi, cudaStream_t s);
// dev_out[c] = largest real active column of panels [c * per, (c + 1) * per), -1 if none
hrpb_status_t chunk_maxcol(const hrpb_handle* h, int64_t per, int nchunks, int* dev_out, cudaStream_t s);

int num_sms();
// NEXT-4: row permutation (degree buckets descending, then min-hash of the column set) and the permuted CSR
hrpb_status_t reorder_impl(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                           const float* values, int32_t* perm, int64_t* row_ptr_out, int32_t* col_idx_out,
                           float* values_out, cudaStream_t s);

// per-device one-time initialisation (kernel attributes, pools): true the first time it is called for the current
// device with this flag word (always true on device ids >= 64)
bool first_on_device(std::atomic<uint64_t>& done);
// records that `s` read the handle (hrpb_spmm on a stream other than the build stream)
void note_use(hrpb_handle* h, cudaStream_t s);

// (tm, tk) pairs the builder and the SpMM both implement: tm in {16, 32, 64, 128} with tk = 16, tm in {16, 32, 64}
// with tk = 32 (the decoder's brick-slot table has one lane per brick: (tm / 16) (tk / 4) <= 32)
inline bool tile_supported(int32_t tm, int32_t tk) {
  return (tk == 16 && (tm == 16 || tm == 32 || tm == 64 || tm == 128)) || (tk == 32 && (tm == 16 || tm == 32 || tm == 64));
}

}  // namespace hrpb
