// internal.h — library-internal declarations shared by api.cu, build.cu and spmm.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hrpb.h"

struct hrpb_handle {
  int64_t M, K, nnz, P, NB, bytes;
  int32_t tm, tk;
  uint32_t* brp;    // [P+1]
  uint32_t* ac;     // [NB_cap * tk]
  uint64_t* sp;     // [NB_cap + 1]
  uint8_t* packed;  // [bytes_cap]
  cudaStream_t stream;  // build stream (frees are ordered on it)
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
// synchronizes s, returns INVALID_CSR if any sticky build (sticky = true above) flagged its input since the
// last call, and clears the flag
hrpb_status_t sticky_take(cudaStream_t s);

hrpb_status_t spmm_impl(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, cudaStream_t s);
// C rows of panels [p_lo, p_hi) only (the pipelined host entry point)
hrpb_status_t spmm_range_impl(const hrpb_handle* h, const float* B, int64_t ldb, float* C, int64_t N, int64_t p_lo,
                              int64_t p_hi, cudaStream_t s);
// dev_out[c] = largest real active column of panels [c * per, (c + 1) * per), -1 if none
hrpb_status_t chunk_maxcol(const hrpb_handle* h, int64_t per, int nchunks, int* dev_out, cudaStream_t s);

int num_sms();

}  // namespace hrpb
