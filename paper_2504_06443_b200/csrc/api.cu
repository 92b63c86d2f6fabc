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

bool first_on_device(std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return true;
  const uint64_t bit = 1ull << dev;
  return (done.fetch_or(bit) & bit) == 0;
}

static void keep_pool_memory() {
  static std::atomic<uint64_t> done{0};
  if (!first_on_device(done)) return;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~0ull;  // keep freed blocks cached in the stream-ordered pool
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
}

static std::mutex g_use_mu;

void note_use(hrpb_handle* h, cudaStream_t s) {
  if (!h || s == h->stream) return;
  std::lock_guard<std::mutex> lk(g_use_mu);
  int i = 0;
  while (i < h->n_use && h->use_st[i] != s) ++i;
  if (i == h->n_use) {
    if (i == hrpb_handle::kMaxUse || cudaEventCreateWithFlags(&h->use_ev[i], cudaEventDisableTiming) != cudaSuccess) {
      h->use_overflow = true;
      return;
    }
    h->use_st[i] = s;
    ++h->n_use;
  }
  cudaEventRecord(h->use_ev[i], s);
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

int num_sms() {  // cached per device (called on every launch)
  static int cached[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && cached[dev] > 0) return cached[dev];
  int n = 148;
  cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  n = n > 0 ? n : 148;
  if (dev >= 0 && dev < 64) cached[dev] = n;
  return n;
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
  {
    std::lock_guard<std::mutex> lk(g_use_mu);
    // SpMMs on other streams may still read the arrays: order the frees after them
    if (h->use_overflow) cudaDeviceSynchronize();
    for (int i = 0; i < h->n_use; ++i) {
      cudaStreamWaitEvent(s, h->use_ev[i], 0);
      cudaEventDestroy(h->use_ev[i]);
    }
    h->n_use = 0;
  }
  dfree(h->brp, s);
  dfree(h->ac, s);
  dfree(h->sp, s);
  dfree(h->packed, s);
  delete h;
}

static bool valid_tile(int32_t tm, int32_t tk) { return tm == 0 ? (tk == 16 || tk == 32) : tile_supported(tm, tk); }

// tm == 0: automatic choice (choose_tm) for the CSR on the device
static hrpb_status_t resolve_tm(int64_t M, int64_t K, int64_t nnz, const int64_t* rp, const int32_t* ci, int32_t tm,
                                int32_t tk, cudaStream_t s, int32_t* out) {
  *out = tm;
  if (tm != 0) return HRPB_SUCCESS;
  hrpb_status_t st = choose_tm(M, K, nnz, rp, ci, s, out, nullptr);
  if (st == HRPB_SUCCESS && tk == 32 && *out > 64) *out = 64;
  return st;
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
  const int32_t tm_req = cfg ? cfg->tm : 16, tk = cfg ? cfg->tk : 16;
  if (!valid_tile(tm_req, tk)) return HRPB_ERROR_INVALID_VALUE;
  hrpb_status_t st = check_device();
  if (st != HRPB_SUCCESS) return st;
  int32_t tm = tm_req;
  st = resolve_tm(M, K, nnz, row_ptr, col_idx, tm_req, tk, (cudaStream_t)stream, &tm);
  if (st != HRPB_SUCCESS) return st;
  hrpb_handle* h = new (std::nothrow) hrpb_handle();
  if (!h) return HRPB_ERROR_OUT_OF_MEMORY;
  st = build_impl(M, K, nnz, row_ptr, col_idx, values, tm, tk, (cudaStream_t)stream, h);
  if (st != HRPB_SUCCESS) {
    release(h);
    return st;
  }
  *out = h;
  return HRPB_SUCCESS;
}

// Replay plan of hrpb_build_spmm: the second consecutive call with the same arguments (and no handle requested)
// captures the whole enqueue sequence — allocations, builder kernels, size read-back, SpMM kernels, frees —
// into a CUDA graph; later identical calls launch the graph (one host call instead of ~40 API calls, and no
// per-kernel launch latency between the dependent kernels). Any change of arguments falls back to eager calls.
namespace {
struct BuildSpmmPlan {
  int64_t M = -1, K = -1, N = -1, nnz = -1;
  const void *rp = nullptr, *ci = nullptr, *va = nullptr, *B = nullptr, *C = nullptr;
  int32_t tm = -1, tk = 0;  // tm as requested (0 = automatic)
  int32_t tm_res = 0;       // automatic TM resolved on the first call of this key (a planning decision, like the graph)
  cudaStream_t s = nullptr;
  int dev = -1;
  int hits = 0;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;  // launches recorded while capturing (hrpb_launch_count accounting of replays)
  bool same(int64_t M_, int64_t K_, int64_t N_, int64_t nnz_, const void* rp_, const void* ci_, const void* va_,
            const void* B_, const void* C_, int32_t tm_, int32_t tk_, cudaStream_t s_, int dev_) const {
    return M == M_ && K == K_ && N == N_ && nnz == nnz_ && rp == rp_ && ci == ci_ && va == va_ && B == B_ &&
           C == C_ && tm == tm_ && tk == tk_ && s == s_ && dev == dev_;
  }
};
}  // namespace

// enqueue: (ev0) build (deferred read-back into `info`) (ev1) SpMM (ev2); `release_arrays` frees the handle's
// arrays on the stream too (graph capture: the graph owns every allocation it makes)
static hrpb_status_t enqueue_build_spmm(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr,
                                        const int32_t* col_idx, const float* values, const float* B, float* C,
                                        int32_t tm, int32_t tk, cudaStream_t s, hrpb_handle* h, uint64_t* info,
                                        cudaEvent_t* ev, bool capturing, bool release_arrays) {
  const unsigned fl = capturing ? cudaEventRecordExternal : 0u;
  cudaEventRecordWithFlags(ev[0], s, fl);
  // inside a graph the build also ORs its status into the sticky word (replays may be asynchronous)
  hrpb_status_t st = build_impl(M, K, nnz, row_ptr, col_idx, values, tm, tk, s, h, info, capturing);
  cudaEventRecordWithFlags(ev[1], s, fl);
  // the SpMM goes in right behind the build (no host round trip between them); it reads the HRPB arrays on
  // the device, so it does not need the sizes the build reports
  if (st == HRPB_SUCCESS && M > 0 && N > 0) st = spmm_impl(h, B, N, C, N, s);
  cudaEventRecordWithFlags(ev[2], s, fl);
  if (release_arrays) {
    dfree(h->brp, s); dfree(h->ac, s); dfree(h->sp, s); dfree(h->packed, s);
    h->brp = nullptr; h->ac = nullptr; h->sp = nullptr; h->packed = nullptr;
  }
  return st;
}

// pinned read-back buffer, phase events (per device: an event records only on streams of its own device) and the
// replay plan: one set per host thread
static thread_local uint64_t* t_info = nullptr;
static thread_local cudaEvent_t t_ev_dev[64][3];
static thread_local cudaEvent_t* t_ev = nullptr;  // the events of this thread's most recent build_spmm call

static cudaEvent_t* device_events() {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return nullptr;
  cudaEvent_t* ev = t_ev_dev[dev];
  if (!ev[0])
    for (int i = 0; i < 3; ++i)
      if (cudaEventCreate(&ev[i]) != cudaSuccess) return nullptr;
  return ev;
}

static hrpb_status_t build_spmm_common(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr,
                                       const int32_t* col_idx, const float* values, const float* B, float* C,
                                       const hrpb_config_t* cfg, hrpb_stream_t stream, hrpb_t* out,
                                       float* phase_ms, bool async) {
  if (out) *out = nullptr;
  if (M < 0 || K < 0 || N < 0 || nnz < 0 || M >= (1ll << 31) || K >= (1ll << 31) || N >= (1ll << 31) || !row_ptr)
    return HRPB_ERROR_INVALID_VALUE;
  if ((nnz > 0 && (!col_idx || !values)) || (M > 0 && N > 0 && !C) || (K > 0 && N > 0 && !B))
    return HRPB_ERROR_INVALID_VALUE;
  const int32_t tm_req = cfg ? cfg->tm : 16, tk = cfg ? cfg->tk : 16;
  if (!valid_tile(tm_req, tk)) return HRPB_ERROR_INVALID_VALUE;
  hrpb_status_t st = check_device();
  if (st != HRPB_SUCCESS) return st;
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0;
  cudaGetDevice(&dev);
  static thread_local BuildSpmmPlan plan;
  static thread_local hrpb_handle plan_h;
  if (!t_info && cudaMallocHost(&t_info, 4 * sizeof(uint64_t)) != cudaSuccess) return HRPB_ERROR_OUT_OF_MEMORY;
  cudaEvent_t* ev = device_events();
  if (!ev) return HRPB_ERROR_CUDA;
  t_ev = ev;
  uint64_t* info = t_info;
  static const bool use_graph = [] {
    const char* e = getenv("HRPB_NO_GRAPH");  // debugging aid: always run eagerly
    return !(e && atoi(e));
  }();
  const bool same = plan.same(M, K, N, nnz, row_ptr, col_idx, values, B, C, tm_req, tk, s, dev);
  int32_t tm = tm_req;
  if (same && tm_req == 0 && plan.tm_res > 0) {
    tm = plan.tm_res;
  } else {
    st = resolve_tm(M, K, nnz, row_ptr, col_idx, tm_req, tk, s, &tm);
    if (st != HRPB_SUCCESS) return st;
  }
  if (!out && use_graph && same && plan.hits >= 1) {
    if (!plan.exec) {  // capture the enqueue sequence once
      plan_h = hrpb_handle();
      const int64_t l0 = g_launches.load();
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
      hrpb_status_t cst = HRPB_ERROR_CUDA;
      if (e == cudaSuccess) {
        cst = enqueue_build_spmm(M, K, N, nnz, row_ptr, col_idx, values, B, C, tm, tk, s, &plan_h, info, ev, true,
                                 true);
        e = cudaStreamEndCapture(s, &g);
      }
      if (e == cudaSuccess && cst == HRPB_SUCCESS && g) e = cudaGraphInstantiate(&plan.exec, g, 0);
      if (g) cudaGraphDestroy(g);
      if (e != cudaSuccess || cst != HRPB_SUCCESS) {
        cudaGetLastError();
        plan.exec = nullptr;
        plan.hits = -1000000;  // do not retry this key: eager calls from now on
      }
      plan.kernels = g_launches.load() - l0;
      g_launches.fetch_sub(plan.kernels);  // counted per replay below
    }
    if (plan.exec) {
      cudaError_t e = cudaGraphLaunch(plan.exec, s);
      g_launches.fetch_add(plan.kernels);
      if (async) return e == cudaSuccess ? HRPB_SUCCESS : cuda_status(e);  // status: hrpb_sync_status
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      if (e != cudaSuccess) return cuda_status(e);
      hrpb_handle tmp = hrpb_handle();
      st = build_finish(&tmp, info, HRPB_SUCCESS);
      if (st == HRPB_ERROR_INVALID_CSR) sticky_take(s);  // reported here: not again by hrpb_sync_status
      if (phase_ms && st == HRPB_SUCCESS) {
        cudaEventElapsedTime(&phase_ms[0], ev[0], ev[1]);
        cudaEventElapsedTime(&phase_ms[1], ev[1], ev[2]);
      }
      return st;
    }
  }
  if (!same) {
    if (plan.exec) cudaGraphExecDestroy(plan.exec);
    plan = BuildSpmmPlan();
    plan.M = M; plan.K = K; plan.N = N; plan.nnz = nnz; plan.rp = row_ptr; plan.ci = col_idx; plan.va = values;
    plan.B = B; plan.C = C; plan.tm = tm_req; plan.tk = tk; plan.s = s; plan.dev = dev;
    plan.tm_res = tm;
  }
  ++plan.hits;
  hrpb_handle* h = new (std::nothrow) hrpb_handle();
  if (!h) return HRPB_ERROR_OUT_OF_MEMORY;
  st = enqueue_build_spmm(M, K, N, nnz, row_ptr, col_idx, values, B, C, tm, tk, s, h, info, ev, false, false);
  const cudaError_t e = cudaStreamSynchronize(s);
  if (st == HRPB_SUCCESS && e != cudaSuccess) st = cuda_status(e);
  if (st == HRPB_SUCCESS) st = build_finish(h, info, st);  // INVALID_CSR is reported here (C is then undefined)
  if (phase_ms && st == HRPB_SUCCESS) {
    cudaEventElapsedTime(&phase_ms[0], ev[0], ev[1]);
    cudaEventElapsedTime(&phase_ms[1], ev[1], ev[2]);
  }
  if (st != HRPB_SUCCESS || !out) {
    release(h);
    return st;
  }
  *out = h;
  return HRPB_SUCCESS;
}

hrpb_status_t hrpb_build_spmm(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr,
                              const int32_t* col_idx, const float* values, const float* B, float* C,
                              const hrpb_config_t* cfg, hrpb_stream_t stream, hrpb_t* out, float* phase_ms) {
  return build_spmm_common(M, K, N, nnz, row_ptr, col_idx, values, B, C, cfg, stream, out, phase_ms, false);
}

hrpb_status_t hrpb_build_spmm_async(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr,
                                    const int32_t* col_idx, const float* values, const float* B, float* C,
                                    const hrpb_config_t* cfg, hrpb_stream_t stream) {
  return build_spmm_common(M, K, N, nnz, row_ptr, col_idx, values, B, C, cfg, stream, nullptr, nullptr, true);
}

hrpb_status_t hrpb_sync_status(hrpb_stream_t stream, float* phase_ms) {
  hrpb_status_t st = check_device();
  if (st != HRPB_SUCCESS) return st;
  st = sticky_take((cudaStream_t)stream);
  if (phase_ms && st == HRPB_SUCCESS && t_ev) {
    cudaEventElapsedTime(&phase_ms[0], t_ev[0], t_ev[1]);
    cudaEventElapsedTime(&phase_ms[1], t_ev[1], t_ev[2]);
  }
  return st;
}

hrpb_status_t hrpb_spmm(const hrpb_t A, const float* B, float* C, int64_t M, int64_t K, int64_t N,
                        hrpb_stream_t stream) {
  if (!A || N < 0) return HRPB_ERROR_INVALID_VALUE;
  if (M != A->M || K != A->K) return HRPB_ERROR_DIMENSION_MISMATCH;
  if (N == 0 || M == 0) return HRPB_SUCCESS;
  if (!C || (!B && K > 0)) return HRPB_ERROR_INVALID_VALUE;
  if (N >= (1ll << 31)) return HRPB_ERROR_INVALID_VALUE;
  const hrpb_status_t st = spmm_impl(A, B, N, C, N, (cudaStream_t)stream);
  if (st == HRPB_SUCCESS) note_use(A, (cudaStream_t)stream);
  return st;
}

hrpb_status_t hrpb_spmm_sharded(const hrpb_t A, const float* const* shards, int32_t nshards, int64_t rows_per_shard,
                                float* C, int64_t M, int64_t K, int64_t N, hrpb_stream_t stream) {
  if (!A || N < 0 || !shards) return HRPB_ERROR_INVALID_VALUE;
  if (M != A->M || K != A->K) return HRPB_ERROR_DIMENSION_MISMATCH;
  if (N >= (1ll << 31)) return HRPB_ERROR_INVALID_VALUE;
  if (N == 0 || M == 0) return HRPB_SUCCESS;
  if (!C) return HRPB_ERROR_INVALID_VALUE;
  const hrpb_status_t st = spmm_sharded_impl(A, shards, nshards, rows_per_shard, C, N, (cudaStream_t)stream);
  if (st == HRPB_SUCCESS) note_use(A, (cudaStream_t)stream);
  return st;
}

hrpb_status_t hrpb_reorder_rows(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                                const float* values, int32_t* perm, int64_t* row_ptr_out, int32_t* col_idx_out,
                                float* values_out, hrpb_stream_t stream) {
  if (M < 0 || K < 0 || nnz < 0 || M >= (1ll << 31) || nnz >= (1ll << 31) || !row_ptr || !row_ptr_out ||
      (M > 0 && !perm) || (nnz > 0 && (!col_idx || !values || !col_idx_out || !values_out)))
    return HRPB_ERROR_INVALID_VALUE;
  hrpb_status_t st = check_device();
  if (st != HRPB_SUCCESS) return st;
  return reorder_impl(M, K, nnz, row_ptr, col_idx, values, perm, row_ptr_out, col_idx_out, values_out,
                      (cudaStream_t)stream);
}

hrpb_status_t hrpb_set_row_map(hrpb_t A, const int32_t* row_map) {
  if (!A) return HRPB_ERROR_INVALID_VALUE;
  A->row_map = row_map;
  return HRPB_SUCCESS;
}

hrpb_status_t hrpb_build_spmm_host(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr_h,
                                   const int32_t* col_idx_h, const float* values_h, const float* B_h, float* C_h,
                                   const hrpb_config_t* cfg, hrpb_stream_t stream) {
  if (M < 0 || K < 0 || N < 0 || nnz < 0 || !row_ptr_h || (nnz > 0 && (!col_idx_h || !values_h)) ||
      (M > 0 && N > 0 && !C_h) || (K > 0 && N > 0 && !B_h))
    return HRPB_ERROR_INVALID_VALUE;
  if (M >= (1ll << 31) || K >= (1ll << 31) || N >= (1ll << 31)) return HRPB_ERROR_INVALID_VALUE;
  if (!valid_tile(cfg ? cfg->tm : 16, cfg ? cfg->tk : 16)) return HRPB_ERROR_INVALID_VALUE;
  hrpb_status_t st = check_device();
  if (st != HRPB_SUCCESS) return st;
  cudaStream_t s = (cudaStream_t)stream;
  // Pipeline: copy engine H2D: CSR, then B in row chunks; the build runs as soon as the CSR is in;
  // C is produced in panel chunks, chunk c starting once the B rows up to its largest active column have
  // arrived; its rows go back D2H on a third stream while later B chunks still stream in (PCIe is full duplex).
  // library copy streams, one pair per device (a stream belongs to the device current at its creation)
  static cudaStream_t s_h2d_dev[64], s_d2h_dev[64];
  static std::mutex s_mu;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64) return HRPB_ERROR_NOT_SUPPORTED;
  cudaStream_t s_h2d, s_d2h;
  {
    std::lock_guard<std::mutex> lk(s_mu);
    if (!s_h2d_dev[dev]) {
      cudaStreamCreateWithFlags(&s_h2d_dev[dev], cudaStreamNonBlocking);
      cudaStreamCreateWithFlags(&s_d2h_dev[dev], cudaStreamNonBlocking);
    }
    s_h2d = s_h2d_dev[dev];
    s_d2h = s_d2h_dev[dev];
  }
#ifndef HRPB_E2E_BCH
#define HRPB_E2E_BCH 32
#define HRPB_E2E_CCH 16
#endif
  constexpr int kBChunks = HRPB_E2E_BCH, kCChunks = HRPB_E2E_CCH;
  cudaEvent_t ev[2 + kBChunks + kCChunks];
  for (auto& x : ev) cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
  cudaEvent_t ev_in = ev[0], ev_done = ev[1], *ev_b = ev + 2, *ev_c = ev + 2 + kBChunks;
  int64_t* rp = (int64_t*)dalloc((M + 1) * sizeof(int64_t), s);
  int32_t* ci = (int32_t*)dalloc((nnz + 1) * sizeof(int32_t), s);
  float* v = (float*)dalloc((nnz + 1) * sizeof(float), s);
  float* B = (float*)dalloc((size_t)K * N * sizeof(float) + 16, s);
  float* C = (float*)dalloc((size_t)M * N * sizeof(float) + 16, s);
  int* maxcol = (int*)dalloc(kCChunks * sizeof(int), s);
  int maxcol_h[kCChunks];
  hrpb_t A = nullptr;
  if (!rp || !ci || !v || !B || !C || !maxcol) st = HRPB_ERROR_OUT_OF_MEMORY;
  cudaError_t e = cudaSuccess;
  auto ok = [&](cudaError_t x) {
    if (x != cudaSuccess && e == cudaSuccess) e = x;
  };
  const int64_t brows = (K + kBChunks - 1) / kBChunks;  // B rows per H2D chunk
  if (st == HRPB_SUCCESS) {
    ok(cudaEventRecord(ev_in, s));  // the allocations above are ordered on s
    ok(cudaStreamWaitEvent(s_h2d, ev_in, 0));
    ok(cudaMemcpyAsync(rp, row_ptr_h, (M + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, s_h2d));
    if (nnz) ok(cudaMemcpyAsync(ci, col_idx_h, nnz * sizeof(int32_t), cudaMemcpyHostToDevice, s_h2d));
    if (nnz) ok(cudaMemcpyAsync(v, values_h, nnz * sizeof(float), cudaMemcpyHostToDevice, s_h2d));
    ok(cudaEventRecord(ev_in, s_h2d));
    for (int j = 0; j < kBChunks; ++j) {
      const int64_t r0 = j * brows, r1 = (j + 1) * brows < K ? (j + 1) * brows : K;
      if (r1 > r0 && N > 0)
        ok(cudaMemcpyAsync(B + r0 * N, B_h + r0 * N, (size_t)(r1 - r0) * N * sizeof(float), cudaMemcpyHostToDevice,
                           s_h2d));
      ok(cudaEventRecord(ev_b[j], s_h2d));
    }
    ok(cudaStreamWaitEvent(s, ev_in, 0));
    if (e != cudaSuccess) st = cuda_status(e);
  }
  if (st == HRPB_SUCCESS) st = hrpb_build(M, K, nnz, rp, ci, v, cfg, stream, &A);  // (syncs s, not the copies)
  const int64_t P = A ? A->P : 0;
  const int64_t per = (P + kCChunks - 1) / kCChunks > 0 ? (P + kCChunks - 1) / kCChunks : 1;
  if (st == HRPB_SUCCESS && M > 0 && N > 0) st = chunk_maxcol(A, per, kCChunks, maxcol, s);
  if (st == HRPB_SUCCESS && M > 0 && N > 0) {
    ok(cudaMemcpyAsync(maxcol_h, maxcol, sizeof(maxcol_h), cudaMemcpyDeviceToHost, s));
    ok(cudaStreamSynchronize(s));
    if (e != cudaSuccess) st = cuda_status(e);
  }
  if (st == HRPB_SUCCESS && M > 0 && N > 0) {
    if (N % 4 != 0) {  // padded-B path of the kernel: whole-matrix launch after all of B
      ok(cudaStreamWaitEvent(s, ev_b[kBChunks - 1], 0));
      st = hrpb_spmm(A, B, C, M, K, N, stream);
      ok(cudaEventRecord(ev_c[0], s));
      ok(cudaStreamWaitEvent(s_d2h, ev_c[0], 0));
      ok(cudaMemcpyAsync(C_h, C, (size_t)M * N * sizeof(float), cudaMemcpyDeviceToHost, s_d2h));
    } else {
      int waited = -1;
      for (int c = 0; c < kCChunks && st == HRPB_SUCCESS; ++c) {
        const int64_t p0 = c * per, p1 = (c + 1) * per < P ? (c + 1) * per : P;
        if (p1 <= p0) break;
        const int need = maxcol_h[c] < 0 ? -1 : (int)(maxcol_h[c] / brows);  // last B chunk this C chunk reads
        if (need > waited) {
          ok(cudaStreamWaitEvent(s, ev_b[need], 0));
          waited = need;
        }
        st = spmm_range_impl(A, B, N, C, N, p0, p1, s);
        ok(cudaEventRecord(ev_c[c], s));
        const int64_t r0 = p0 * A->tm, r1 = p1 * A->tm < M ? p1 * A->tm : M;
        ok(cudaStreamWaitEvent(s_d2h, ev_c[c], 0));
        ok(cudaMemcpyAsync(C_h + r0 * N, C + r0 * N, (size_t)(r1 - r0) * N * sizeof(float), cudaMemcpyDeviceToHost,
                           s_d2h));
      }
    }
    if (e != cudaSuccess && st == HRPB_SUCCESS) st = cuda_status(e);
  }
  // every stream drains before the buffers are released on s
  cudaEventRecord(ev_done, s_h2d);
  cudaStreamWaitEvent(s, ev_done, 0);
  cudaEventRecord(ev_done, s_d2h);
  cudaStreamWaitEvent(s, ev_done, 0);
  hrpb_free(A);
  dfree(rp, s); dfree(ci, s); dfree(v, s); dfree(B, s); dfree(C, s); dfree(maxcol, s);
  cudaError_t e2 = cudaStreamSynchronize(s);
  if (st == HRPB_SUCCESS && e2 != cudaSuccess) st = cuda_status(e2);
  for (auto& x : ev) cudaEventDestroy(x);
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
