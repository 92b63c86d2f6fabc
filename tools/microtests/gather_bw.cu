// Gather-bandwidth microbenchmark for the SpMM B-row staging (SURVEY §7 microtest T6).
// Every CTA (1 per SM) streams R "blocks" of 16 random rows x ROWB bytes from a row-major matrix
// into a ring of D shared-memory stages and a consumer warp frees stages as they complete.
// method 0: cp.async 16 B (LDGSTS), 4 producer warps (block-parallel), noinc arrive
// method 1: TMA tile::gather4 (box 32 fp32, SWIZZLE_128B_ATOM_32B), 1 thread per producer warp
// method 2: LDG.128 -> STS by producer lanes, then mbarrier arrive
// method 3: cp.async.bulk 1-D (ROWB bytes per row), 1 thread per producer warp
// Prints aggregate GB/s of gathered bytes. Rows: uniform over `nrows_window` (L2-resident if small).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(2);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" :: "r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
}

constexpr int kWarpsProd = 4;
__device__ __forceinline__ const void* dst_base_dummy(const void* p) { return p; }
constexpr int kThreads = 32 * (kWarpsProd + 1);

template <int METHOD, int ROWB>
__global__ void __launch_bounds__(kThreads, 1)
gather(const __grid_constant__ CUtensorMap tm, const float* __restrict__ B, int ncols, const uint32_t* __restrict__ rows,
       int nblk, int D, unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  constexpr int kStage = 16 * ROWB;
  uint64_t* full = (uint64_t*)(sm + (size_t)D * kStage);
  uint64_t* empty = full + D;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < D; ++s) {
      mbar_init(&full[s], METHOD == 0 || METHOD == 2 || METHOD == 4 ? 32 : 1);
      mbar_init(&empty[s], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t* myrows = rows + (size_t)blockIdx.x * nblk * 16;
  if (warp < kWarpsProd) {
    int s = warp % D;
    uint32_t ph = (warp / D) & 1;
    for (int i = warp; i < nblk; i += kWarpsProd) {
      mbar_wait(&empty[s], ph ^ 1);
      uint8_t* dst = sm + (size_t)s * kStage;
      const uint32_t rl = myrows[i * 16 + (lane & 15)];
      if (METHOD == 0) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint32_t rk = __shfl_sync(0xffffffffu, rl, r);
          const float* src = B + (size_t)rk * ncols;
#pragma unroll
          for (int c = lane; c < ROWB / 16; c += 32)
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + r * ROWB + c * 16)),
                         "l"(src + 4 * c) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
      } else if (METHOD == 4) {
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint32_t rk = __shfl_sync(0xffffffffu, rl, r);
          const float* src = B + (size_t)rk * ncols;
#pragma unroll
          for (int c = lane; c < ROWB / 16; c += 32) {
            const uint32_t at = c >> 3, g = (c >> 1) & 3, rq = r & 3;
            const uint32_t d = su32(dst) + (r >> 2) * (ROWB / 128) * 512 + at * 512 + rq * 128 +
                               ((g ^ rq) << 5) + ((c & 1) << 4);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src + 4 * c),
                         "r"(rk < 0xFFFFFFF0u ? 16u : 0u) : "memory");
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
      } else if (METHOD == 1) {
        uint32_t rr[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) rr[r] = __shfl_sync(0xffffffffu, rl, r);
        if (lane == 0) {
          mbar_expect_tx(&full[s], 16 * ROWB);
#pragma unroll
          for (int g = 0; g < 4; ++g)
#pragma unroll
            for (int a = 0; a < ROWB / 128; ++a)
              asm volatile(
                  "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
                  " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(su32(dst + (g * (ROWB / 128) + a) * 512)),
                  "l"(&tm), "r"(32 * a), "r"(rr[4 * g]), "r"(rr[4 * g + 1]), "r"(rr[4 * g + 2]), "r"(rr[4 * g + 3]),
                  "r"(su32(&full[s]))
                  : "memory");
        }
      } else if (METHOD == 2) {
        float4 v[16 * ROWB / 512];
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const uint32_t rk = __shfl_sync(0xffffffffu, rl, r);
#pragma unroll
          for (int c = 0; c < ROWB / 512; ++c)
            v[r * (ROWB / 512) + c] = __ldcg(reinterpret_cast<const float4*>(B + (size_t)rk * ncols) + lane + 32 * c);
        }
#pragma unroll
        for (int r = 0; r < 16; ++r)
#pragma unroll
          for (int c = 0; c < ROWB / 512; ++c)
            *reinterpret_cast<float4*>(dst + r * ROWB + (lane + 32 * c) * 16) = v[r * (ROWB / 512) + c];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&full[s]);
      } else {
        uint32_t rr[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) rr[r] = __shfl_sync(0xffffffffu, rl, r);
        if (lane == 0) {
          mbar_expect_tx(&full[s], 16 * ROWB);
#pragma unroll
          for (int r = 0; r < 16; ++r)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    su32(dst + r * ROWB)),
                "l"(B + (size_t)rr[r] * ncols), "r"(ROWB), "r"(su32(&full[s]))
                : "memory");
        }
      }
      __syncwarp();
      s += kWarpsProd;
      if (s >= D) { s -= D; ph ^= 1; }
    }
  } else {
    unsigned long long acc = 0;
    int s = 0;
    uint32_t ph = 0;
    for (int i = 0; i < nblk; ++i) {
      mbar_wait(&full[s], ph);
      acc += *reinterpret_cast<const uint32_t*>(sm + (size_t)s * kStage + lane * 4);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (++s == D) { s = 0; ph ^= 1; }
    }
    if (acc == 0x12345) sink[0] = acc;
  }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int M, int ROWB>
float run(const CUtensorMap& tm, const float* B, int ncols, const uint32_t* rows, int nblk, int D, int grid,
          unsigned long long* sink) {
  size_t smem = 1024 + (size_t)D * 16 * ROWB + 2 * D * 8;
  CK(cudaFuncSetAttribute(gather<M, ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gather<M, ROWB><<<grid, kThreads, smem>>>(tm, B, ncols, rows, nblk, D, sink);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 3; ++it) gather<M, ROWB><<<grid, kThreads, smem>>>(tm, B, ncols, rows, nblk, D, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 3;
}

int main(int argc, char** argv) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  const int ncols = 128;  // 512-B rows
  const size_t total_rows = 1 << 20;
  float* B;
  CK(cudaMalloc(&B, total_rows * ncols * 4));
  CK(cudaMemset(B, 0, total_rows * ncols * 4));
  const int nblk = 2048;
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)ncols, (cuuint64_t)total_rows};
  cuuint64_t gstr[1] = {(cuuint64_t)ncols * 4};
  cuuint32_t box[2] = {32, 1}, es[2] = {1, 1};
  ((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, B, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                 CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  std::vector<uint32_t> file_rows;
  if (argc > 1) {  // real activeCols replay: uint32 [nsm][nblk][16], sentinel rows mapped to row 0
    FILE* f = fopen(argv[1], "rb");
    file_rows.resize((size_t)nsm * nblk * 16);
    size_t got = fread(file_rows.data(), 4, file_rows.size(), f);
    fclose(f);
    printf("replaying %zu rows from %s\n", got, argv[1]);
  }
  for (int window : {1 << 14, 1 << 20, -1, -2}) {  // 8 MB (L2), 512 MB (DRAM), banded c2a-like, file
    if (window == -2 && file_rows.empty()) continue;
    std::vector<uint32_t> h((size_t)nsm * nblk * 16);
    if (window == -2) h = file_rows;
    srand(1);
    if (window > 0) {
      for (auto& x : h) x = (uint32_t)(((uint64_t)rand() * 2654435761ull) % window);
    } else {  // CTA c walks panels p = c*P/nsm ..: ~5 blocks per panel of 16 sorted rows in [16p-32, 16p+48)
      for (int c = 0; c < nsm; ++c)
        for (int i = 0; i < nblk; ++i) {
          int64_t p = (int64_t)c * 65536 / nsm + i / 5;
          for (int r = 0; r < 16; ++r) {
            int64_t v = 16 * p - 32 + (rand() % 80);
            if (v < 0) v = 0;
            h[((size_t)c * nblk + i) * 16 + r] = (uint32_t)(v % (1 << 20));
          }
        }
    }
    uint32_t* rows;
    CK(cudaMalloc(&rows, h.size() * 4));
    CK(cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    const double bytes = (double)nsm * nblk * 16 * 512;
    for (int D : {8, 16}) {
      float t0 = run<0, 512>(tm, B, ncols, rows, nblk, D, nsm, sink);
      float t1 = run<1, 512>(tm, B, ncols, rows, nblk, D, nsm, sink);
      float t2 = run<2, 512>(tm, B, ncols, rows, nblk, D, nsm, sink);
      float t3 = run<3, 512>(tm, B, ncols, rows, nblk, D, nsm, sink);
      float t4 = run<4, 512>(tm, B, ncols, rows, nblk, D, nsm, sink);
      printf("window %8d rows  D=%2d  cp.async %7.0f | gather4 %7.0f | ldg+sts %7.0f | bulk1d %7.0f | cp.async-zfill-swz %7.0f GB/s\n",
             window, D, bytes / t0 / 1e6, bytes / t1 / 1e6, bytes / t2 / 1e6, bytes / t3 / 1e6, bytes / t4 / 1e6);
    }
    cudaFree(rows);
  }
  return 0;
}
