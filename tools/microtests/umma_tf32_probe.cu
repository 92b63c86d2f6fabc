// Microtest T1/T2/T3/T4 (SURVEY.md §7 "Microtests to run on the box first").
//
// One CTA, 128 threads. It stages a 16-row x (2 x 128)-column slice of a dense
// row-major matrix with TMA tile::gather4 (SWIZZLE_128B, MN-major UMMA operand),
// writes a 16x16 "decoded block" as a K-major no-swizzle UMMA operand (four
// 16x4 bricks, row-major inside a brick), runs tcgen05.mma.kind::tf32 with
// M=128 (dense width), N=16 (panel rows), K=8 x 2, and reads TMEM back.
//
//   T3: layout/descriptor check against a CPU product.
//   T4: sentinel row index (== K, out of bounds) and columns >= N zero-fill.
//   T1: TF32 operand conversion: truncation or round-to-nearest.
//   T2: FP32 accumulation in TMEM stays exact for integers below 2^24.
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o probe umma_tf32_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cmath>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); exit(2);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t par) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(su32(b)), "r"(par) : "memory");
  }
}
__device__ __forceinline__ void gather4(void* dst, const CUtensorMap* tm, int c0, int r0, int r1, int r2, int r3,
                                        uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
      :: "r"(su32(dst)), "l"(tm), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm100)
  d |= (uint64_t)(layout & 7) << 61;
  return d;
}
__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t idesc, uint32_t acc) {
  asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p; }"
               :: "r"(dt), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
}

// idesc: D=F32, A=B=TF32, A MN-major, B K-major, N=16, M=128.
constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (1u << 15) | (0u << 16) | ((16u >> 3) << 17) |
                           ((128u >> 4) << 24);

struct Params {
  const float* Atile;  // [16][16] row-major: A_block[r][k]
  const int* rows;     // [16] B rows to gather (== K means sentinel)
  float* C;            // [16][ncols]
  int ncols;           // padded output width (256)
  int reps;            // extra accumulate repetitions (T2)
  const float* Atile2; // tile used for the repetitions
};

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tm, Params p) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  float* btile = (float*)smem;                 // 2 kgroups x 8 atoms x 1 KB = 16 KB
  float* atile = (float*)(smem + 16384);       // 1 KB
  float* atile2 = (float*)(smem + 16384 + 1024);
  uint64_t* bars = (uint64_t*)(smem + 16384 + 2048);
  uint32_t* tslot = (uint32_t*)(bars + 4);
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;

  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(su32(tslot)), "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  // A^T tile: brick bc = k/4 holds 16 rows x 4 cols row-major (bit order of the HRPB pattern).
  for (int i = tid; i < 256; i += 128) {
    int r = i / 16, k = i % 16;
    atile[(k / 4) * 64 + r * 4 + (k % 4)] = p.Atile[r * 16 + k];
    atile2[(k / 4) * 64 + r * 4 + (k % 4)] = p.Atile2[r * 16 + k];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = *tslot;

  if (tid == 0) {
    mbar_expect_tx(&bars[0], 16 * 8 * 128);
    for (int g4 = 0; g4 < 4; ++g4)
      for (int a = 0; a < 8; ++a) {
        uint8_t* dst = smem + (g4 * 8 + a) * 512;
        const int* r = p.rows + 4 * g4;
        gather4(dst, &tm, 32 * a, r[0], r[1], r[2], r[3], &bars[0]);
      }
    mbar_wait(&bars[0], 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    for (int t = 0; t < 2; ++t)
      for (int g = 0; g < 2; ++g) {
        uint64_t ad = sdesc(su32(smem + (2 * g * 8 + 4 * t) * 512), 512, 8 * 512, 1);
        uint64_t bd = sdesc(su32(atile) + g * 512, 256, 128, 0);
        mma_tf32(tbase + t * 16, ad, bd, IDESC, g > 0);
      }
    for (int rep = 0; rep < p.reps; ++rep)
      for (int t = 0; t < 2; ++t)
        for (int g = 0; g < 2; ++g) {
          uint64_t ad = sdesc(su32(smem + (2 * g * 8 + 4 * t) * 512), 512, 8 * 512, 1);
          uint64_t bd = sdesc(su32(atile2) + g * 512, 256, 128, 0);
          mma_tf32(tbase + t * 16, ad, bd, IDESC, 1);
        }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(su32(&bars[1]))
                 : "memory");
  }
  __syncwarp();
  mbar_wait(&bars[1], 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int t = 0; t < 2; ++t) {
    uint32_t v[16];
    uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + t * 16;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    int n = t * 128 + 32 * warp + lane;
    for (int r = 0; r < 16; ++r) p.C[r * p.ncols + n] = __uint_as_float(v[r]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tbase), "r"(32));
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeFn get_encode() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  return (EncodeFn)fn;
}

struct Case {
  const char* name;
  int K, N;  // gathered matrix K x N (row-major, ld = N)
  std::vector<float> B, A, A2;
  std::vector<int> rows;
  int reps;
};

static int run_case(Case& c, EncodeFn enc, bool print_all) {
  const int NC = 256;
  float *dB, *dA, *dA2, *dC;
  int* dR;
  CK(cudaMalloc(&dB, c.B.size() * 4));
  CK(cudaMalloc(&dA, 256 * 4));
  CK(cudaMalloc(&dA2, 256 * 4));
  CK(cudaMalloc(&dC, 16 * NC * 4));
  CK(cudaMalloc(&dR, 16 * 4));
  CK(cudaMemcpy(dB, c.B.data(), c.B.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dA, c.A.data(), 256 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dA2, c.A2.data(), 256 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dR, c.rows.data(), 16 * 4, cudaMemcpyHostToDevice));
  CK(cudaMemset(dC, 0xFF, 16 * NC * 4));
  CUtensorMap tm;
  cuuint64_t gdim[2] = {(cuuint64_t)c.N, (cuuint64_t)c.K};
  cuuint64_t gstr[1] = {(cuuint64_t)c.N * 4};
  cuuint32_t box[2] = {32, 1};
  cuuint32_t es[2] = {1, 1};
  CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dB, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) { printf("[%s] encode failed %d\n", c.name, (int)r); return 1; }
  Params p{dA, dR, dC, NC, c.reps, dA2};
  size_t smem = 16384 + 2048 + 64 + 1024;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  probe<<<1, 128, smem>>>(tm, p);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<float> C(16 * NC);
  CK(cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost));
  // CPU expectation (exact operand values; fp64 accumulate)
  int bad = 0;
  double maxerr = 0;
  for (int rr = 0; rr < 16; ++rr)
    for (int n = 0; n < NC; ++n) {
      double s = 0;
      for (int k = 0; k < 16; ++k) {
        int row = c.rows[k];
        double b = (row < c.K && n < c.N) ? c.B[(size_t)row * c.N + n] : 0.0;
        s += (double)c.A[rr * 16 + k] * b + (double)c.reps * (double)c.A2[rr * 16 + k] * b;
      }
      double e = fabs(s - (double)C[rr * NC + n]);
      if (e > maxerr) maxerr = e;
      if (e > 1e-3 * (1 + fabs(s))) {
        if (bad < 8) printf("[%s] mismatch r=%d n=%d got %.9g want %.9g\n", c.name, rr, n, C[rr * NC + n], s);
        ++bad;
      }
    }
  printf("[%s] %s  max|err|=%.3g  C[0][0]=%.9g C[1][5]=%.9g\n", c.name, bad ? "FAIL" : "PASS", maxerr, C[0], C[NC + 5]);
  if (print_all) {
    printf("[%s] C[0][0..3] = %.10g %.10g %.10g %.10g\n", c.name, C[0], C[1], C[2], C[3]);
  }
  cudaFree(dB); cudaFree(dA); cudaFree(dA2); cudaFree(dC); cudaFree(dR);
  return bad ? 1 : 0;
}

int main() {
  EncodeFn enc = get_encode();
  int fails = 0;
  srand(12345);
  {  // T3 + T4: random integers, a sentinel row, N = 200 (columns 200..255 OOB).
    Case c;
    c.name = "T3T4-layout";
    c.K = 64; c.N = 200;
    c.B.resize((size_t)c.K * c.N);
    for (auto& x : c.B) x = (float)(rand() % 9 - 4);
    c.A.resize(256); c.A2.assign(256, 0.f);
    for (auto& x : c.A) x = (float)(rand() % 7 - 3);
    c.rows = {3, 17, 0, 63, 5, 5, 40, 22, 9, 64 /*sentinel*/, 11, 12, 50, 33, 2, 64 /*sentinel*/};
    c.reps = 0;
    fails += run_case(c, enc, false);
  }
  {  // T3 with non-integer values.
    Case c;
    c.name = "T3-float";
    c.K = 4096; c.N = 256;
    c.B.resize((size_t)c.K * c.N);
    for (auto& x : c.B) x = (float)rand() / RAND_MAX - 0.5f;
    c.A.resize(256); c.A2.assign(256, 0.f);
    for (auto& x : c.A) x = (float)rand() / RAND_MAX - 0.5f;
    for (int i = 0; i < 16; ++i) c.rows.push_back(rand() % c.K);
    c.reps = 0;
    fails += run_case(c, enc, false);
  }
  {  // T1: A = 1 + 2^-11 + 2^-12 against B = 1 (A is the K-major UMMA operand).
    Case c;
    c.name = "T1-roundA";
    c.K = 16; c.N = 256;
    c.B.assign((size_t)c.K * c.N, 0.f);
    for (int n = 0; n < c.N; ++n) c.B[n] = 1.0f;  // row 0 = 1
    c.A.assign(256, 0.f); c.A2.assign(256, 0.f);
    for (int r = 0; r < 16; ++r) c.A[r * 16 + 0] = 1.0f + ldexpf(1, -11) + ldexpf(1, -12);
    c.rows = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15};
    c.reps = 0;
    run_case(c, enc, true);  // informative: 1.0 => truncation, 1.0009765625 => RN
  }
  {  // T1: B = 1 + 2^-11 + 2^-12 against A = 1 (B is the gathered MN-major operand).
    Case c;
    c.name = "T1-roundB";
    c.K = 16; c.N = 256;
    c.B.assign((size_t)c.K * c.N, 0.f);
    for (int n = 0; n < c.N; ++n) c.B[n] = 1.0f + ldexpf(1, -11) + ldexpf(1, -12);
    c.A.assign(256, 0.f); c.A2.assign(256, 0.f);
    for (int r = 0; r < 16; ++r) c.A[r * 16 + 0] = 1.0f;
    c.rows = {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15};
    c.reps = 0;
    run_case(c, enc, true);
  }
  {  // T2: start at 2^23 (2^11 * 2^12), then add +1 per repetition: exact iff FP32 accumulation is exact.
    Case c;
    c.name = "T2-exact-accum";
    c.K = 16; c.N = 256;
    c.B.assign((size_t)c.K * c.N, 0.f);
    for (int n = 0; n < c.N; ++n) { c.B[n] = 4096.0f; c.B[c.N + n] = 1.0f; }
    c.A.assign(256, 0.f); c.A2.assign(256, 0.f);
    for (int r = 0; r < 16; ++r) { c.A[r * 16 + 0] = 2048.0f; c.A2[r * 16 + 1] = 1.0f; }
    c.rows = {0, 1, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15, 15};
    c.reps = 3000;
    fails += run_case(c, enc, true);
  }
  printf("probe done, hard failures: %d\n", fails);
  return fails ? 1 : 0;
}
