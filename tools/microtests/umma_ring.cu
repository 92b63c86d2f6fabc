// tcgen05.mma.kind::tf32 issue pattern of the SpMM MMA warp: per "block" G MMAs (M = 128, N = 16, K = 8) into
// NT accumulator tiles, then tcgen05.commit to the block's stage barrier (ring of S stages); before block i the
// issuer waits for the commit of block i - S (the producer's empty wait folded into the issuer). Cycles per block.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46) | ((uint64_t)(layout & 7) << 61);
}
__device__ __forceinline__ void wait_par(uint64_t* b, uint32_t ph) {
  uint32_t ok = 0;
  for (long long it = 0; !ok && it < 20000000ll; ++it)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su32(b)), "r"(ph) : "memory");
}

template <int N, int M>
__global__ void ring(int R, int S, int G, int NTT, int commit_every, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm_raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)sm_raw + 1023) & ~(uintptr_t)1023);
  __shared__ uint64_t bar[32];
  __shared__ uint32_t tslot;
  const int warp = threadIdx.x / 32;
  for (int i = threadIdx.x; i < 16384; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (threadIdx.x == 0) {
    for (int s = 0; s < 32; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
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
    // M = 128: A = gathered rows MN-major SW128_32B, N = panel rows; M = 64: A = panel tile K-major, N = dense cols
    const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((M == 128 ? 1u : 0u) << 15) |
                           ((M == 128 ? 0u : 1u) << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
    const uint64_t ad = M == 128 ? sdesc(su32(sm), 512, 2048, 1) : sdesc(su32(sm + 32768), 1024, 128, 0);
    const uint64_t bd = M == 128 ? sdesc(su32(sm + 32768), N * 16, 128, 0) : sdesc(su32(sm), 512, 2048, 1);
    long long t0 = clock64();
    for (int i = 0; i < R; ++i) {
      if (i >= S && (i % commit_every) == 0) wait_par(&bar[(i / commit_every) % S], ((i / commit_every - S) / S) & 1);
      for (int g = 0; g < G; ++g)
        for (int t = 0; t < NTT; ++t)
          asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                       ::"r"(tb + (uint32_t)(t * N)), "l"(ad), "l"(bd), "r"(idesc), "r"(g) : "memory");
      if ((i + 1) % commit_every == 0)
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                     ::"r"(su32(&bar[(i / commit_every) % S])));
    }
    long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(512));
}

template <int N, int M>
void run(const char* name, int S, int G, int NTT, int ce = 1) {
  long long* d;
  cudaMalloc(&d, 16);
  const int R = 8000;
  cudaFuncSetAttribute(ring<N, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70 * 1024);
  ring<N, M><<<148, 128, 70 * 1024>>>(R, S, G, NTT, ce, d);
  cudaDeviceSynchronize();
  long long h[1];
  cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
  fflush(stdout); printf("%-26s S %2d MMAs/block %d commit/%d blocks: %7.1f cyc/block (%s)\n", name, S, G * NTT, ce, (double)h[0] / R,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
  fflush(stdout);
}

int main() {
  for (int S : {4, 8, 12, 20}) run<16, 128>("M128 N16 K8 (transposed)", S, 2, 2);
  for (int S : {4, 12}) run<16, 128>("M128 N16 K8 (transposed)", S, 2, 1);
  run<16, 128>("M128 N16 K8 (transposed)", 12, 2, 2, 2);
  run<16, 128>("M128 N16 K8 (transposed)", 12, 2, 2, 4);
  run<16, 128>("M128 N16 K8 no wait", 1 << 20, 2, 2, 1);
  for (int S : {4, 12}) run<256, 64>("M64 N256 K8 (direct)", S, 2, 1);
  for (int S : {4, 12}) run<128, 64>("M64 N128 K8 (direct)", S, 2, 1);
  run<256, 64>("M64 N256 K8 no wait", 1 << 20, 2, 1);
  return 0;
}
