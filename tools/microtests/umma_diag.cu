// Diagnostic for tcgen05.mma.kind::tf32 operand descriptors (see umma_tf32_probe.cu).
// mode 0: A (M=128 x K=8) K-major no-swizzle, B (K=8 x N=16) K-major no-swizzle, both written by threads.
// mode 1: A MN-major no-swizzle written by threads, B K-major no-swizzle.
// mode 2: A MN-major SW128 written by threads (manual swizzle), B K-major no-swizzle.
// Each mode first pre-fills TMEM with 7.0 via tcgen05.st, then runs one MMA with accumulate=flag.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(2);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}

__global__ void __launch_bounds__(128, 1) diag(int mode, int acc, const float* A /*[128][8] A[m][k]*/,
                                               const float* B /*[8][16] B[k][n]*/, float* D /*[128][16]*/,
                                               uint32_t idesc_override) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* sa = (float*)smem;            // 4 KB (128 x 8 fp32)
  float* sb = (float*)(smem + 4096);   // 512 B (8 x 16)
  uint64_t* bar = (uint64_t*)(smem + 8192);
  uint32_t* tslot = (uint32_t*)(smem + 8192 + 64);
  int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  if (tid == 0) { mbar_init(bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(tslot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // fill A
  for (int i = tid; i < 128 * 8; i += 128) {
    int m = i / 8, k = i % 8;
    float v = A[m * 8 + k];
    uint32_t off;
    if (mode == 0) {  // K-major interleave: core (8 rows x 16B); SBO(m-group)=128, LBO(k-group)=2048
      off = (m % 8) * 16 + (k % 4) * 4 + (m / 8) * 128 + (k / 4) * 2048;
    } else if (mode == 1) {  // MN-major interleave: core (8 k-rows x 16B of 4 m); SBO(m-group of 4)=128, LBO(k-grp)
      off = (m % 4) * 4 + (k % 8) * 16 + (m / 4) * 128;
    } else if (mode == 2) {  // MN-major SW128: atom 32 m x 8 k, row k at k*128, 16B chunk XOR k; atoms (m/32) at LBO=1024
      uint32_t lin = (k % 8) * 128 + (m % 32) * 4;
      uint32_t chunk = (lin >> 4) & 7, row = (lin >> 7) & 7;
      lin = (lin & ~(7u << 4)) | ((chunk ^ row) << 4);
      off = (m / 32) * 1024 + lin;
    } else {  // MN-major SW128_BASE32B: atom 32 m x 4 k (512 B), 32B chunk XOR (k%4); atoms (m/32) LBO=512, k-grp SBO=2048
      uint32_t lin = (k % 4) * 128 + (m % 32) * 4;
      uint32_t chunk = (lin >> 5) & 3, row = (lin >> 7) & 3;
      lin = (lin & ~(3u << 5)) | ((chunk ^ row) << 5);
      off = (m / 32) * 512 + (k / 4) * 2048 + lin;
    }
    *(float*)((uint8_t*)sa + off) = v;
  }
  for (int i = tid; i < 8 * 16; i += 128) {  // B K-major interleave: (n,k): (n%8)*16+(k%4)*4+(n/8)*SBO(128)+(k/4)*LBO(256)
    int k = i / 16, n = i % 16;
    uint32_t off = (n % 8) * 16 + (k % 4) * 4 + (n / 8) * 128 + (k / 4) * 256;
    *(float*)((uint8_t*)sb + off) = B[k * 16 + n];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t tbase = *tslot;
  // prefill TMEM with 7.0
  {
    uint32_t s = __float_as_uint(7.0f);
    uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16);
    asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
                 :: "r"(taddr), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s),
                    "r"(s), "r"(s), "r"(s), "r"(s), "r"(s), "r"(s) : "memory");
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    uint32_t a_major = mode == 0 ? 0u : 1u;
    uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | (a_major << 15) | (0u << 16) | ((16u >> 3) << 17) |
                     ((128u >> 4) << 24);
    if (idesc_override) idesc = idesc_override | (a_major << 15);
    uint64_t ad;
    if (mode == 0) ad = sdesc(su32(sa), 2048, 128, 0);
    else if (mode == 1) ad = sdesc(su32(sa), 4096 /*unused k-group*/, 128, 0);
    else if (mode == 2) ad = sdesc(su32(sa), 1024, 8192, 2);
    else ad = sdesc(su32(sa), 512, 2048, 1);
    uint64_t bd = sdesc(su32(sb), 256, 128, 0);
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
                 :: "r"(tbase), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(bar))
                 : "memory");
  }
  __syncwarp();
  mbar_wait(bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[16];
  uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  int m = 32 * warp + lane;
  for (int n = 0; n < 16; ++n) D[m * 16 + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "r"(32));
}

int main() {
  std::vector<float> A(128 * 8), B(8 * 16), D(128 * 16);
  srand(7);
  for (auto& x : A) x = (float)(rand() % 7 - 3);
  for (auto& x : B) x = (float)(rand() % 5 - 2);
  float *dA, *dB, *dD;
  CK(cudaMalloc(&dA, A.size() * 4)); CK(cudaMalloc(&dB, B.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaFuncSetAttribute(diag, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384));
  for (int mode = 0; mode < 4; ++mode)
    for (int acc = 0; acc < 2; ++acc) {
      CK(cudaMemset(dD, 0xFF, D.size() * 4));
      diag<<<1, 128, 16384>>>(mode, acc, dA, dB, dD, 0);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
      int bad = 0, n7 = 0;
      for (int m = 0; m < 128; ++m)
        for (int n = 0; n < 16; ++n) {
          double s = acc ? 7.0 : 0.0;
          for (int k = 0; k < 8; ++k) s += (double)A[m * 8 + k] * B[k * 16 + n];
          if (D[m * 16 + n] == 7.0f) ++n7;
          if (fabs(s - D[m * 16 + n]) > 1e-3) ++bad;
        }
      printf("mode %d acc %d: %s bad=%d  (#==7.0: %d)  D[0][0..3]=%g %g %g %g\n", mode, acc, bad ? "FAIL" : "PASS",
             bad, n7, D[0], D[1], D[2], D[3]);
    }
  return 0;
}
