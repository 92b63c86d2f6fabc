// Cost of tcgen05.commit in an MMA stream: one thread issues R groups of m MMAs (M = 128, N = 16, K = 8, TF32),
// each group followed by tcgen05.commit to one of 8 mbarriers (no waits); then waits for the last commit.
// Reports issue and completion cycles per group. m = 0: commits only.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)(layout & 7) << 61);
}

__global__ void kcommit(int R, int m, int nthreads_issue, int nch, int NN, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[16];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 16; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tb = tslot;
  // issuing threads: lane 0 of warps 0 .. nthreads_issue - 1 (each its own 8 barriers and accumulators)
  if ((threadIdx.x & 31) == 0 && warp < nthreads_issue) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | ((uint32_t)(NN >> 3) << 17) |
                           ((128u >> 4) << 24);
    const uint64_t ad = sdesc(su32(sm), 512, 2048, 1);
    const uint64_t bd = sdesc(su32(sm + 32768), 256, 128, 0);
    uint64_t* mb = bar + 8 * warp;
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      for (int j = 0; j < m; ++j)
        asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                     ::"r"(tb + (uint32_t)(256 * warp + NN * ((i * m + j) % nch))), "l"(ad), "l"(bd), "r"(idesc), "r"(i > 0 ? 1 : 0) : "memory");
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&mb[i & 7])));
    }
    long long t1 = clock64();
    // last commit: group R - 1 on barrier (R - 1) & 7, its ((R - 1) >> 3)-th completion
    const uint32_t par = ((R - 1) >> 3) & 1;
    uint32_t ok = 0;
    for (long long it = 0; !ok && it < 50000000ll; ++it)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(su32(&mb[(R - 1) & 7])), "r"(par) : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0 && warp == 0) { out[0] = t1 - t0; out[1] = t2 - t0; out[2] = ok; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

int main() {
  long long* d;
  cudaMalloc(&d, 32);
  cudaFuncSetAttribute(kcommit, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  int cfg[][4] = {{1, 4, 1, 16}, {1, 4, 2, 16}, {1, 4, 4, 16}, {1, 4, 8, 16}, {1, 4, 16, 16}, {2, 4, 2, 16}, {2, 4, 8, 16},
                  {1, 8, 8, 16}, {1, 8, 16, 16}, {1, 2, 1, 64}, {1, 2, 2, 64}, {1, 2, 4, 64}, {1, 4, 4, 32}, {1, 4, 8, 32}};
  for (auto& c : cfg) {
      const int nt = c[0], m = c[1], nch = c[2], NN = c[3];
      const int R = 8000;  // multiple of 16: the last barrier's completion count is even/odd as computed
      kcommit<<<148, 64, 70 * 1024>>>(R, m, nt, nch, NN, d);
      cudaError_t e = cudaDeviceSynchronize();
      long long h[3];
      cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
      printf("N %3d chains %2d issuers %d  MMAs/commit %2d: issue %7.1f cyc/group, complete %7.1f cyc/group  ok %lld (%s)\n", NN, nch, nt, m,
             (double)h[0] / R, (double)h[1] / R, h[2], cudaGetErrorString(e));
      fflush(stdout);
    }
  return 0;
}
