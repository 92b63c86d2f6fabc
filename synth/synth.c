/*
 * synth.c — seeded, counter-based synthetic inputs for the HRPB SpMM tests and bench.
 *
 * This module is shared by BOTH sides of the parity check (the CPU oracle in oracle/
 * and the CUDA path in paper_2504_06443_b200/). It contains none of the method's
 * arithmetic: it only draws canonical CSR matrices (0-based, row_ptr int64, columns
 * strictly increasing within a row) and dense row-major matrices from a seed.
 *
 * Random numbers: h(seed, i) = splitmix64(seed ^ splitmix64(i)), with the counter i
 * built from (row, slot) or (edge, level) so any index range can be regenerated
 * independently (SURVEY.md §8(d) "Synthetic inputs").
 *
 * Structures (recipes stated in DESIGN.md §"Input recipe"):
 *   bernoulli   : keep (i,j) iff h(seed, i*K+j) < p*2^64                     (config 1)
 *   banded      : row i draws d distinct cols uniformly in [i-w, i+w) ∩ [0,K)  (config 2a)
 *   clustered   : panel p (16 rows) gets 4 distinct dense 16x4 clusters at
 *                 col-block (4p + U[-32,32)) mod (K/4)                        (config 2b)
 *   rmat        : Graph500 R-MAT, (a,b,c,d), duplicates removed, optional
 *                 seeded vertex relabelling                                  (config 3)
 *   uniform_d   : d distinct uniform columns per row                          (config 4)
 *   fem         : 2-D grid of nodes, `bs` dofs per node, dense bs x bs blocks on
 *                 the 9-point stencil + 1 random block per block row          (config 5)
 * Values (per stored entry e, or per dense element index):
 *   mode 0 (exact): A in {-2,-1,1,2}[h & 3]; B = (h mod 5) - 2  (TF32-exact integers)
 *   mode 1 (float): (h >> 40) * 2^-23 - 1, uniform on [-1, 1), exact in fp32
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
static inline uint64_t hh(uint64_t seed, uint64_t i) { return splitmix64(seed ^ splitmix64(i)); }
static inline uint64_t hh2(uint64_t seed, uint64_t a, uint64_t b) {
  return hh(seed, a * 0x100000001B3ull + splitmix64(b + 0x632BE59BD9B4E019ull));
}

uint64_t synth_hash(uint64_t seed, uint64_t i) { return hh(seed, i); }

typedef struct {
  int64_t M, K, nnz;
  int64_t* row_ptr;
  int32_t* col_idx;
} synth_csr_t;

void synth_free(void* p) { free(p); }

static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}

/* insertion sort for short rows, qsort otherwise */
static void sort_i32(int32_t* v, int64_t n) {
  if (n < 32) {
    for (int64_t i = 1; i < n; ++i) {
      int32_t x = v[i];
      int64_t j = i - 1;
      while (j >= 0 && v[j] > x) { v[j + 1] = v[j]; --j; }
      v[j + 1] = x;
    }
  } else {
    qsort(v, (size_t)n, sizeof(int32_t), cmp_i32);
  }
}

static int64_t exclusive_scan(int64_t* a, int64_t n) { /* a[0..n] ; a[i] counts -> offsets */
  int64_t s = 0;
  for (int64_t i = 0; i < n; ++i) { int64_t c = a[i]; a[i] = s; s += c; }
  a[n] = s;
  return s;
}

/* ---- per-row "d distinct uniform in [lo,hi)" by rejection ---------------------------------- */
static int64_t draw_distinct(uint64_t seed, int64_t row, int64_t lo, int64_t hi, int64_t d, int32_t* out) {
  int64_t range = hi - lo;
  if (range <= 0) return 0;
  if (d >= range) {
    for (int64_t j = 0; j < range; ++j) out[j] = (int32_t)(lo + j);
    return range;
  }
  int64_t have = 0;
  uint64_t slot = 0;
  while (have < d) {
    int32_t c = (int32_t)(lo + (int64_t)(hh2(seed, (uint64_t)row, slot++) % (uint64_t)range));
    int dup = 0;
    for (int64_t j = 0; j < have; ++j) if (out[j] == c) { dup = 1; break; }
    if (!dup) out[have++] = c;
  }
  sort_i32(out, have);
  return have;
}

static int alloc_csr(synth_csr_t* o, int64_t M, int64_t K) {
  o->M = M; o->K = K; o->nnz = 0;
  o->row_ptr = (int64_t*)calloc((size_t)M + 1, sizeof(int64_t));
  o->col_idx = NULL;
  return o->row_ptr ? 0 : -1;
}

/* banded: rows [r0, r0+M) of the banded matrix (global row index g = r0 + i), so a rank can draw
 * its own row slab of a larger matrix without generating the rest. */
int synth_banded_rows(int64_t r0, int64_t M, int64_t K, int64_t d, int64_t w, int64_t shift, uint64_t seed,
                      synth_csr_t* o) {
  /* row g = r0 + i draws from the band centred at g - shift (shift lets a rank's slab reuse B) */
  if (alloc_csr(o, M, K)) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int64_t g = r0 + i, ctr = g - shift;
    int64_t lo = ctr - w < 0 ? 0 : ctr - w, hi = ctr + w > K ? K : ctr + w;
    int64_t r = hi - lo;
    o->row_ptr[i] = r < 0 ? 0 : (d < r ? d : r);
  }
  int64_t nnz = exclusive_scan(o->row_ptr, M);
  o->nnz = nnz;
  o->col_idx = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  if (!o->col_idx) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int64_t g = r0 + i, ctr = g - shift;
    int64_t lo = ctr - w < 0 ? 0 : ctr - w, hi = ctr + w > K ? K : ctr + w;
    draw_distinct(seed, g, lo, hi, d, o->col_idx + o->row_ptr[i]);
  }
  return 0;
}
int synth_banded(int64_t M, int64_t K, int64_t d, int64_t w, uint64_t seed, synth_csr_t* o) {
  return synth_banded_rows(0, M, K, d, w, 0, seed, o);
}

int synth_uniform_d(int64_t M, int64_t K, int64_t d, uint64_t seed, synth_csr_t* o) {
  if (alloc_csr(o, M, K)) return -1;
  int64_t dd = d < K ? d : K;
  for (int64_t i = 0; i < M; ++i) o->row_ptr[i] = dd;
  int64_t nnz = exclusive_scan(o->row_ptr, M);
  o->nnz = nnz;
  o->col_idx = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  if (!o->col_idx) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) draw_distinct(seed, i, 0, K, dd, o->col_idx + o->row_ptr[i]);
  return 0;
}

int synth_bernoulli(int64_t M, int64_t K, double p, uint64_t seed, synth_csr_t* o) {
  if (alloc_csr(o, M, K)) return -1;
  long double thr_ld = (long double)p * 18446744073709551616.0L;
  uint64_t thr = p >= 1.0 ? UINT64_MAX : (uint64_t)thr_ld;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int64_t c = 0;
    for (int64_t j = 0; j < K; ++j) c += hh(seed, (uint64_t)(i * K + j)) < thr;
    o->row_ptr[i] = c;
  }
  int64_t nnz = exclusive_scan(o->row_ptr, M);
  o->nnz = nnz;
  o->col_idx = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  if (!o->col_idx) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int64_t w = o->row_ptr[i];
    for (int64_t j = 0; j < K; ++j)
      if (hh(seed, (uint64_t)(i * K + j)) < thr) o->col_idx[w++] = (int32_t)j;
  }
  return 0;
}

/* clustered: panel p = rows [16p, 16p+16) gets `ncl` distinct dense 16x4 clusters */
int synth_clustered(int64_t M, int64_t K, int64_t ncl, int64_t spread, uint64_t seed, synth_csr_t* o) {
  if (alloc_csr(o, M, K)) return -1;
  int64_t KB = K / 4; /* column blocks of width 4 */
  int64_t P = (M + 15) / 16;
  if (KB <= 0) { o->col_idx = (int32_t*)malloc(4); return 0; }
  int64_t nc = ncl < KB ? ncl : KB;
  int32_t* cb = (int32_t*)malloc((size_t)(P * nc + 1) * sizeof(int32_t));
  if (!cb) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < P; ++p) {
    int32_t* my = cb + p * nc;
    int64_t have = 0;
    uint64_t slot = 0;
    while (have < nc) {
      int64_t off = (int64_t)(hh2(seed, (uint64_t)p, slot++) % (uint64_t)(2 * spread)) - spread;
      int64_t b = ((4 * p + off) % KB + KB) % KB;
      int dup = 0;
      for (int64_t j = 0; j < have; ++j) if (my[j] == b) { dup = 1; break; }
      if (!dup) my[have++] = (int32_t)b;
    }
    sort_i32(my, nc);
  }
  for (int64_t i = 0; i < M; ++i) o->row_ptr[i] = 4 * nc;
  int64_t nnz = exclusive_scan(o->row_ptr, M);
  o->nnz = nnz;
  o->col_idx = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  if (!o->col_idx) { free(cb); return -1; }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    const int32_t* my = cb + (i / 16) * nc;
    int32_t* dst = o->col_idx + o->row_ptr[i];
    for (int64_t j = 0; j < nc; ++j)
      for (int t = 0; t < 4; ++t) dst[4 * j + t] = 4 * my[j] + t;
  }
  free(cb);
  return 0;
}

/* FEM-like: nodes on an nx x ny grid, bs dofs per node, 9-point stencil + 1 random node block */
int synth_fem(int64_t nx, int64_t ny, int64_t bs, uint64_t seed, synth_csr_t* o) {
  int64_t nodes = nx * ny, M = nodes * bs;
  if (alloc_csr(o, M, M)) return -1;
  int64_t* nbr = (int64_t*)malloc((size_t)nodes * 10 * sizeof(int64_t));
  int32_t* nn = (int32_t*)malloc((size_t)nodes * sizeof(int32_t));
  if (!nbr || !nn) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < nodes; ++v) {
    int64_t x = v % nx, y = v / nx, cnt = 0;
    int64_t* my = nbr + v * 10;
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        int64_t xx = x + dx, yy = y + dy;
        if (xx >= 0 && xx < nx && yy >= 0 && yy < ny) my[cnt++] = yy * nx + xx;
      }
    uint64_t slot = 0;
    for (;;) { /* one random extra block, distinct from the stencil blocks */
      int64_t r = (int64_t)(hh2(seed, (uint64_t)v, slot++) % (uint64_t)nodes);
      int dup = 0;
      for (int64_t j = 0; j < cnt; ++j) if (my[j] == r) { dup = 1; break; }
      if (!dup) { my[cnt++] = r; break; }
      if (cnt >= nodes) break;
    }
    /* sort node ids */
    for (int64_t a = 1; a < cnt; ++a) {
      int64_t t = my[a], b = a - 1;
      while (b >= 0 && my[b] > t) { my[b + 1] = my[b]; --b; }
      my[b + 1] = t;
    }
    nn[v] = (int32_t)cnt;
  }
  for (int64_t i = 0; i < M; ++i) o->row_ptr[i] = (int64_t)nn[i / bs] * bs;
  int64_t nnz = exclusive_scan(o->row_ptr, M);
  o->nnz = nnz;
  o->col_idx = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  if (!o->col_idx) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < M; ++i) {
    int64_t v = i / bs;
    int32_t* dst = o->col_idx + o->row_ptr[i];
    for (int64_t j = 0; j < nn[v]; ++j)
      for (int64_t t = 0; t < bs; ++t) dst[j * bs + t] = (int32_t)(nbr[v * 10 + j] * bs + t);
  }
  free(nbr); free(nn);
  return 0;
}

/* R-MAT (Graph500 style): E = ef * 2^scale edges, each drawn with `scale` quadrant choices. */
int synth_rmat(int64_t scale, int64_t ef, double a, double b, double c, int permute, uint64_t seed,
               synth_csr_t* o) {
  int64_t n = (int64_t)1 << scale, E = ef * n;
  if (alloc_csr(o, n, n)) return -1;
  uint64_t* ek = (uint64_t*)malloc((size_t)E * sizeof(uint64_t));
  if (!ek) return -1;
  const double ab = a + b, abc = a + b + c;
  int64_t* perm = NULL;
  if (permute) { /* seeded Fisher-Yates relabelling of vertex ids (rows and columns alike) */
    perm = (int64_t*)malloc((size_t)n * sizeof(int64_t));
    for (int64_t i = 0; i < n; ++i) perm[i] = i;
    for (int64_t i = n - 1; i > 0; --i) {
      int64_t j = (int64_t)(hh(seed ^ 0x5bd1e995ull, (uint64_t)i) % (uint64_t)(i + 1));
      int64_t t = perm[i]; perm[i] = perm[j]; perm[j] = t;
    }
  }
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < E; ++e) {
    uint64_t r = 0, col = 0;
    for (int64_t l = 0; l < scale; ++l) {
      double u = (double)(hh2(seed, (uint64_t)e, (uint64_t)l) >> 11) * (1.0 / 9007199254740992.0);
      int q = u < a ? 0 : (u < ab ? 1 : (u < abc ? 2 : 3));
      r = (r << 1) | (uint64_t)(q >> 1);
      col = (col << 1) | (uint64_t)(q & 1);
    }
    if (perm) { r = (uint64_t)perm[r]; col = (uint64_t)perm[col]; }
    ek[e] = (r << 32) | col;
  }
  free(perm);
  /* bucket by row (counting sort), then sort + dedupe within each row */
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < E; ++e) cnt[ek[e] >> 32]++;
  exclusive_scan(cnt, n);
  int32_t* tmp = (int32_t*)malloc((size_t)(E ? E : 1) * sizeof(int32_t));
  int64_t* cur = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  memcpy(cur, cnt, (size_t)n * sizeof(int64_t));
  for (int64_t e = 0; e < E; ++e) { uint64_t r = ek[e] >> 32; tmp[cur[r]++] = (int32_t)(ek[e] & 0xFFFFFFFFu); }
  free(ek); free(cur);
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    int32_t* v = tmp + cnt[i];
    int64_t m = cnt[i + 1] - cnt[i];
    sort_i32(v, m);
    int64_t u = 0;
    for (int64_t j = 0; j < m; ++j) if (u == 0 || v[u - 1] != v[j]) v[u++] = v[j];
    o->row_ptr[i] = u;
  }
  int64_t nnz = exclusive_scan(o->row_ptr, n);
  o->nnz = nnz;
  o->col_idx = (int32_t*)malloc((size_t)(nnz ? nnz : 1) * sizeof(int32_t));
  if (!o->col_idx) { free(tmp); free(cnt); return -1; }
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i)
    memcpy(o->col_idx + o->row_ptr[i], tmp + cnt[i], (size_t)(o->row_ptr[i + 1] - o->row_ptr[i]) * sizeof(int32_t));
  free(tmp); free(cnt);
  return 0;
}

/* ---- values ---------------------------------------------------------------------------------- */
/* A values for stored entries [e0, e0+n): mode 0 exact {-2,-1,1,2}, mode 1 float [-1,1) */
void synth_values_a(int64_t e0, int64_t n, int mode, uint64_t seed, float* out) {
  static const float lut[4] = {-2.f, -1.f, 1.f, 2.f};
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    uint64_t h = hh(seed, (uint64_t)(e0 + i));
    out[i] = mode == 0 ? lut[h & 3] : (float)((double)(h >> 40) * (1.0 / 8388608.0) - 1.0);
  }
}
/* dense row-major rows [r0, r0+nr) of a (.. x N) matrix: element index = row*N + col */
void synth_dense(int64_t r0, int64_t nr, int64_t N, int mode, uint64_t seed, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < nr; ++i)
    for (int64_t j = 0; j < N; ++j) {
      uint64_t h = hh(seed, (uint64_t)((r0 + i) * N + j));
      out[i * N + j] = mode == 0 ? (float)((int64_t)(h % 5) - 2)
                                 : (float)((double)(h >> 40) * (1.0 / 8388608.0) - 1.0);
    }
}
int synth_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
