// api.cu — C ABI of libhrpb (include/hrpb.h): argument checks, ownership, error mapping.
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>

#include "common.cuh"
#include "internal.h"

namespace hrpb {

static std::atomic<int64_t> g_launches{0};
static thread_local int g_last_cuda = 0;

void note_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

hrpb_status_t cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return HRPB_SUCCESS;
  g_last_cuda = (int)e;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return HRPB_ERROR_OUT_OF_MEMORY;
  }
  return HRPB_ERROR_CUDA;
}

static void keep_pool_memory() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;  // keep freed blocks cached in the stream-ordered pool
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  });
}

void* dalloc(size_t bytes, cudaStream_t s) {
  keep_pool_memory();
  void* p = nullptr;
  if (cudaMallocAsync(&p, bytes ? bytes : 16, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dfree(void* p, cudaStream_t s) {
  if (p) cudaFreeAsync(p, s);
}

int num_sms() {
  int dev = 0, n = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

static hrpb_status_t check_device() {
  int dev = 0, major = 0, minor = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  if (e != cudaSuccess) return cuda_status(e);
  return (major == 10 && minor == 0) ? HRPB_SUCCESS : HRPB_ERROR_NOT_SUPPORTED;
}

static void release(hrpb_handle* h) {
  if (!h) return;
  cudaStream_t s = h->stream;
  dfree(h->brp, s);
  dfree(h->ac, s);
  dfree(h->sp, s);
  dfree(h->packed, s);
  dfree(h->bpad, s);
  delete h;
}

}  // namespace hrpb

using namespace hrpb;

extern "C" {

hrpb_status_t hrpb_build(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                         const float* values, const hrpb_config_t* cfg, hrpb_stream_t stream, hrpb_t* out) {
  if (!out) return HRPB_ERROR_INVALID_VALUE;
  *out = nullptr;
  if (M < 0 || K < 0 || nnz < 0 || M >= (1ll << 31) || K >= (1ll << 31) || !row_ptr) return HRPB_ERROR_INVALID_VALUE;
  if (nnz > 0 && (!col_idx || !values)) return HRPB_ERROR_INVALID_VALUE;
  const int32_t tm = cfg ? cfg->tm : 16, tk = cfg ? cfg->tk : 16;
  if (!(tm == 16 || tm == 32 || tm == 64 || tm == 128) || !(tk == 16 || tk == 32)) return HRPB_ERROR_INVALID_VALUE;
  hrpb_status_t st = check_device();
  if (st != HRPB_SUCCESS) return st;
  hrpb_handle* h = new (std::nothrow) hrpb_handle;
  if (!h) return HRPB_ERROR_OUT_OF_MEMORY;
  std::memset(h, 0, sizeof(*h));
  st = build_impl(M, K, nnz, row_ptr, col_idx, values, tm, tk, (cudaStream_t)stream, h);
  if (st != HRPB_SUCCESS) {
    release(h);
    return st;
  }
  *out = h;
  return HRPB_SUCCESS;
}

hrpb_status_t hrpb_spmm(const hrpb_t A, const float* B, float* C, int64_t M, int64_t K, int64_t N,
                        hrpb_stream_t stream) {
  if (!A || N < 0) return HRPB_ERROR_INVALID_VALUE;
  if (M != A->M || K != A->K) return HRPB_ERROR_DIMENSION_MISMATCH;
  if (N == 0 || M == 0) return HRPB_SUCCESS;
  if (!C || (!B && K > 0)) return HRPB_ERROR_INVALID_VALUE;
  if (N >= (1ll << 31)) return HRPB_ERROR_INVALID_VALUE;
  return spmm_impl(A, B, N, C, N, (cudaStream_t)stream);
}

hrpb_status_t hrpb_build_spmm_host(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr_h,
                                   const int32_t* col_idx_h, const float* values_h, const float* B_h, float* C_h,
                                   const hrpb_config_t* cfg, hrpb_stream_t stream) {
  if (M < 0 || K < 0 || N < 0 || nnz < 0 || !row_ptr_h || (nnz > 0 && (!col_idx_h || !values_h)) ||
      (M > 0 && N > 0 && !C_h) || (K > 0 && N > 0 && !B_h))
    return HRPB_ERROR_INVALID_VALUE;
  hrpb_status_t st = check_device();
  if (st != HRPB_SUCCESS) return st;
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* rp = (int64_t*)dalloc((M + 1) * sizeof(int64_t), s);
  int32_t* ci = (int32_t*)dalloc((nnz + 1) * sizeof(int32_t), s);
  float* v = (float*)dalloc((nnz + 1) * sizeof(float), s);
  float* B = (float*)dalloc((size_t)K * N * sizeof(float) + 16, s);
  float* C = (float*)dalloc((size_t)M * N * sizeof(float) + 16, s);
  hrpb_t A = nullptr;
  if (!rp || !ci || !v || !B || !C) st = HRPB_ERROR_OUT_OF_MEMORY;
  cudaError_t e = cudaSuccess;
  if (st == HRPB_SUCCESS) {
    e = cudaMemcpyAsync(rp, row_ptr_h, (M + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(ci, col_idx_h, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && nnz) e = cudaMemcpyAsync(v, values_h, nnz * sizeof(float), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess && K * N)
      e = cudaMemcpyAsync(B, B_h, (size_t)K * N * sizeof(float), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) st = cuda_status(e);
  }
  if (st == HRPB_SUCCESS) st = hrpb_build(M, K, nnz, rp, ci, v, cfg, stream, &A);
  if (st == HRPB_SUCCESS) st = hrpb_spmm(A, B, C, M, K, N, stream);
  if (st == HRPB_SUCCESS && M * N) {
    e = cudaMemcpyAsync(C_h, C, (size_t)M * N * sizeof(float), cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) st = cuda_status(e);
  }
  hrpb_free(A);
  dfree(rp, s); dfree(ci, s); dfree(v, s); dfree(B, s); dfree(C, s);
  e = cudaStreamSynchronize(s);
  if (st == HRPB_SUCCESS && e != cudaSuccess) st = cuda_status(e);
  return st;
}

hrpb_status_t hrpb_free(hrpb_t A) {
  release(A);
  return HRPB_SUCCESS;
}

hrpb_status_t hrpb_get_view(const hrpb_t A, hrpb_view_t* v) {
  if (!A || !v) return HRPB_ERROR_INVALID_VALUE;
  v->M = A->M; v->K = A->K; v->nnz = A->nnz;
  v->num_panels = A->P; v->num_blocks = A->NB; v->packed_bytes = A->bytes;
  v->tm = A->tm; v->tk = A->tk;
  v->blockedRowPtr = A->brp; v->activeCols = A->ac; v->sizePtr = A->sp; v->packedBlocks = A->packed;
  return HRPB_SUCCESS;
}

hrpb_status_t hrpb_copy_view_to_host(const hrpb_t A, uint32_t* brp, uint32_t* ac, uint64_t* sp, uint8_t* packed) {
  if (!A) return HRPB_ERROR_INVALID_VALUE;
  cudaError_t e = cudaStreamSynchronize(A->stream);
  if (e == cudaSuccess && brp) e = cudaMemcpy(brp, A->brp, (A->P + 1) * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && ac && A->NB)
    e = cudaMemcpy(ac, A->ac, (size_t)A->NB * A->tk * sizeof(uint32_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && sp) e = cudaMemcpy(sp, A->sp, (A->NB + 1) * sizeof(uint64_t), cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && packed && A->bytes) e = cudaMemcpy(packed, A->packed, A->bytes, cudaMemcpyDeviceToHost);
  return cuda_status(e);
}

const char* hrpb_get_error_string(hrpb_status_t s) {
  switch (s) {
    case HRPB_SUCCESS: return "HRPB_SUCCESS";
    case HRPB_ERROR_INVALID_VALUE: return "HRPB_ERROR_INVALID_VALUE";
    case HRPB_ERROR_INVALID_CSR: return "HRPB_ERROR_INVALID_CSR";
    case HRPB_ERROR_DIMENSION_MISMATCH: return "HRPB_ERROR_DIMENSION_MISMATCH";
    case HRPB_ERROR_OUT_OF_MEMORY: return "HRPB_ERROR_OUT_OF_MEMORY";
    case HRPB_ERROR_NOT_SUPPORTED: return "HRPB_ERROR_NOT_SUPPORTED";
    case HRPB_ERROR_CUDA: return "HRPB_ERROR_CUDA";
  }
  return "HRPB_UNKNOWN_STATUS";
}

int hrpb_last_cuda_error(void) { return g_last_cuda; }

int64_t hrpb_launch_count(void) { return g_launches.load(); }

}  // extern "C"
