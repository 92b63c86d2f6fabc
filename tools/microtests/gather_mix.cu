// Gather microbenchmark for c3-shaped B-row gathers (1-KB rows, N = 256): can a producer keep more bytes in flight
// per SM by splitting a block's 16 rows between the LSU (cp.async) and the bulk-copy engine (cp.async.bulk)?
// Every CTA (1 per SM) streams nblk blocks of 16 rows x ROWB bytes into a ring of D stages; a consumer warp frees
// stages as they complete (the same ring protocol as k_spmm: 4 producer warps, stage i % D).
// method 0: 16 rows by cp.async 16 B (LDGSTS), noinc arrive           (the k_spmm producer)
// method 1: 16 rows by cp.async.bulk (1 instruction per row, lane 0)
// method 2: rows 0..7 cp.async, rows 8..15 cp.async.bulk
// method 3: rows 0..11 cp.async, rows 12..15 cp.async.bulk
// method 4: 16 rows by cp.async with the .L2::256B prefetch-size qualifier
// Row ids: uniform over the window, or R-MAT-like (22 bits, P(bit = 1) = 0.24: c3's column popularity).
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
constexpr int kThreads = 32 * (kWarpsProd + 1);

template <int METHOD, int ROWB>
__global__ void __launch_bounds__(kThreads, 1)
gather(const float* __restrict__ B, int ncols, const uint32_t* __restrict__ rows, int nblk, int D,
       unsigned long long* sink) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  constexpr int kStage = 16 * ROWB;
  constexpr int kLsuRows = METHOD == 1 ? 0 : METHOD == 2 ? 8 : METHOD == 3 ? 12 : 16;
  uint64_t* full = (uint64_t*)(sm + (size_t)D * kStage);
  uint64_t* empty = full + D;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (threadIdx.x == 0) {
    for (int s = 0; s < D; ++s) {
      mbar_init(&full[s], (kLsuRows > 0 ? 32 : 0) + (kLsuRows < 16 ? 1 : 0));
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
      uint32_t rr[16];
#pragma unroll
      for (int r = 0; r < 16; ++r) rr[r] = __shfl_sync(0xffffffffu, rl, r);
      if (kLsuRows < 16 && lane == 0) {
        mbar_expect_tx(&full[s], (16 - kLsuRows) * ROWB);
#pragma unroll
        for (int r = kLsuRows; r < 16; ++r)
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                       ::"r"(su32(dst + r * ROWB)), "l"(B + (size_t)rr[r] * ncols), "r"(ROWB), "r"(su32(&full[s]))
                       : "memory");
      }
      if (kLsuRows > 0) {
#pragma unroll
        for (int r = 0; r < kLsuRows; ++r) {
          const float* src = B + (size_t)rr[r] * ncols;
#pragma unroll
          for (int c = lane; c < ROWB / 16; c += 32) {
            if (METHOD == 4)
              asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(su32(dst + r * ROWB + c * 16)),
                           "l"(src + 4 * c) : "memory");
            else
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + r * ROWB + c * 16)),
                           "l"(src + 4 * c) : "memory");
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
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

template <int M, int ROWB>
float run(const float* B, int ncols, const uint32_t* rows, int nblk, int D, int grid, unsigned long long* sink) {
  size_t smem = 1024 + (size_t)D * 16 * ROWB + 2 * D * 8;
  CK(cudaFuncSetAttribute(gather<M, ROWB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  gather<M, ROWB><<<grid, kThreads, smem>>>(B, ncols, rows, nblk, D, sink);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int it = 0; it < 3; ++it) gather<M, ROWB><<<grid, kThreads, smem>>>(B, ncols, rows, nblk, D, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / 3;
}

int main(int argc, char** argv) {
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  constexpr int ROWB = 1024;
  const int ncols = ROWB / 4;
  const size_t total_rows = 1 << 22;  // c3: K = 4M rows of 1 KB (4 GB)
  float* B;
  CK(cudaMalloc(&B, total_rows * ncols * 4));
  CK(cudaMemset(B, 0, total_rows * ncols * 4));
  const int nblk = 4096;
  unsigned long long* sink;
  CK(cudaMalloc(&sink, 8));
  for (int dist = 0; dist < 4; ++dist) {  // 0: uniform in 16K rows (L2), 1: uniform over 4M, 2: R-MAT popularity,
                                          // 3: replay of a dump_rows.py file (argv[1]: uint32 [nsm][nblk][16])
    if (dist == 3 && argc < 2) break;
    std::vector<uint32_t> h((size_t)nsm * nblk * 16);
    srand(1);
    if (dist == 3) {
      FILE* f = fopen(argv[1], "rb");
      const size_t got = fread(h.data(), 4, h.size(), f);
      fclose(f);
      printf("replaying %zu rows from %s\n", got, argv[1]);
    }
    for (auto& x : h) {
      if (dist == 3) break;
      if (dist == 0) x = (uint32_t)(((uint64_t)rand() * 2654435761ull) % (1 << 14));
      else if (dist == 1) x = (uint32_t)(((uint64_t)rand() * 2654435761ull) % total_rows);
      else {
        uint32_t v = 0;
        for (int b = 0; b < 22; ++b) v |= (uint32_t)((rand() % 100) < 24) << b;
        x = v;
      }
    }
    uint32_t* rows;
    CK(cudaMalloc(&rows, h.size() * 4));
    CK(cudaMemcpy(rows, h.data(), h.size() * 4, cudaMemcpyHostToDevice));
    const double bytes = (double)nsm * nblk * 16 * ROWB;
    for (int D : {8, 12}) {
      const float t0 = run<0, ROWB>(B, ncols, rows, nblk, D, nsm, sink);
      const float t1 = run<1, ROWB>(B, ncols, rows, nblk, D, nsm, sink);
      const float t2 = run<2, ROWB>(B, ncols, rows, nblk, D, nsm, sink);
      const float t3 = run<3, ROWB>(B, ncols, rows, nblk, D, nsm, sink);
      const float t4 = run<4, ROWB>(B, ncols, rows, nblk, D, nsm, sink);
      printf("%-14s D=%2d  cp.async %6.0f | bulk %6.0f | 8+8 %6.0f | 12+4 %6.0f | cp.async.L2::256B %6.0f GB/s\n",
             dist == 0 ? "uniform-L2" : dist == 1 ? "uniform-4M" : dist == 2 ? "rmat-4M" : "replay", D, bytes / t0 / 1e6, bytes / t1 / 1e6,
             bytes / t2 / 1e6, bytes / t3 / 1e6, bytes / t4 / 1e6);
    }
    cudaFree(rows);
  }
  return 0;
}
