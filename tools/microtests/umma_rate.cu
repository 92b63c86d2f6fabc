// tcgen05.mma.kind::tf32 issue/completion rate for the SpMM shapes: M = 128, N = TM in {16, 64},
// K = 8, A (gathered rows) MN-major SWIZZLE_128B_BASE32B vs K-major SWIZZLE_NONE, B K-major.
// One CTA per SM; one thread issues R MMAs back to back, then commits; cycles per MMA via clock64.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)(layout & 7) << 61);
}

template <int N, int AMAJ>
__global__ void rate(int R, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
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
  if (threadIdx.x == 0) {
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)AMAJ << 15) | (0u << 16) |
                           ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t ad = AMAJ ? sdesc(su32(sm), 512, 2048, 1) : sdesc(su32(sm), 2048, 128, 0);
    const uint64_t bd = sdesc(su32(sm + 32768), N * 16, 128, 0);
    long long t0 = clock64();
    for (int r = 0; r < R; ++r) {  // nacc independent accumulators (TMEM columns tb + k N), round robin
      asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                   ::"r"(tb + (uint32_t)((r % nacc) * N)), "l"(ad), "l"(bd), "r"(idesc), "r"((int)(r >= nacc)) : "memory");
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)));
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                   : "=r"(ok) : "r"(su32(&bar)) : "memory");
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N, int AMAJ>
void run(const char* name, int nacc = 1) {
  long long* d;
  cudaMalloc(&d, 16);
  const int R = 20000;
  cudaFuncSetAttribute(rate<N, AMAJ>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  rate<N, AMAJ><<<148, 128, 70 * 1024>>>(R, nacc, d);
  cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-32s acc %d  issue %6.1f cyc/MMA, complete %6.1f cyc/MMA  (%s)\n", name, nacc, (double)h[0] / R, (double)h[1] / R,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int a : {1, 2, 4, 8}) run<16, 1>("M128 N16 K8 A=MN SW128_32B", a);
  for (int a : {1, 2, 4}) run<64, 1>("M128 N64 K8 A=MN SW128_32B", a);
  run<16, 0>("M128 N16 K8 A=K  none");
  run<64, 1>("M128 N64 K8 A=MN SW128_32B");
  run<64, 0>("M128 N64 K8 A=K  none");
  run<128, 1>("M128 N128 K8 A=MN SW128_32B");
  return 0;
}
