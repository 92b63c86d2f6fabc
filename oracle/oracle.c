/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for HRPB SpMM (arxiv 2504.06443).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_2504_06443_b200/) never
 * links, imports or calls anything here, and this file shares no code, header, table or helper
 * with it. Inputs come from synth/ (seeded generators with none of the method's arithmetic).
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn, S:Lnnn = SPEC.md line nnn.
 *
 *  O1 oracle_csr_validate      canonical CSR
 *  O2 oracle_csr_spmm_f64      C = A.B in FP64, ascending CSR order, plus S = sum |a||b|
 *     oracle_csr_spmm_f32out   same arithmetic, fp32 output, all rows, OpenMP (timed CPU baseline)
 *  O3 oracle_dense_gemm_f64    dense triple loop (textbook GEMM) for tiny matrices
 *  O4 oracle_hrpb_convert      CSR -> HRPB, step by step per P:L81-149 (Alg. "CSR to HRPB"
 *                              Phase 1/2), P:L160-167 (§HRPB data structure), with the readings
 *                              R1-R13, R23 of DESIGN.md and the HRPB-v1 byte layout
 *  O5 oracle_hrpb_to_csr       inverse of O4
 *  O6 oracle_hrpb_check        HRPB invariants (north star)
 *  O7 oracle_hrpb_spmm_f64     FP64 SpMM walking HRPB like Alg. "cuTeSpMM kernel design"
 *                               with zero-filled bricks (debug aid)
 *
 * HRPB-v1 block byte layout (reading R7): block b starts at sizePtr[b] (multiple of 16):
 *   u8 colPtr[TK/4 + 1] | u8 rows[nbr] | zero pad to 8 | u64 patterns[nbr] (LE) |
 *   f32 values[nz] | zero pad to 16.
 * Bricks are 16 x 4 (brick_m = 16, brick_k = 4). Pattern bit i (LSB = 0) is the
 * row-major element (i / 4, i % 4) of the brick (reading R3).
 *
 * Parity pins: every function here is pinned by tests/test_oracle.py against things other than
 * itself (brute force, closed forms, SPEC worked examples, round trips); see DESIGN.md §Oracle.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <stdio.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define BRICK_M 16
#define BRICK_K 4

/* ---------------------------------------------------------------- O1: CSR validation */
/* returns 0 if canonical; 1 row_ptr[0]!=0, 2 non-monotone, 3 row_ptr[M]!=nnz, 4 col out of
 * range, 5 columns not strictly increasing in a row */
int oracle_csr_validate(int64_t M, int64_t K, int64_t nnz, const int64_t* rp, const int32_t* ci) {
  if (rp[0] != 0) return 1;
  for (int64_t i = 0; i < M; ++i)
    if (rp[i + 1] < rp[i]) return 2;
  if (rp[M] != nnz) return 3;
  for (int64_t i = 0; i < M; ++i)
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      if (ci[e] < 0 || ci[e] >= K) return 4;
      if (e > rp[i] && ci[e] <= ci[e - 1]) return 5;
    }
  return 0;
}

/* ---------------------------------------------------------------- O2: CSR SpMM in FP64 */
/* C[i][j] = sum_{k in row i} (double)a_ik * (double)b_kj, in ascending CSR order.
 * rows == NULL -> all M rows; otherwise the listed rows, outputs packed [nrows][N].
 * S (optional) = sum |a_ik| |b_kj| (the float-mode tolerance scale). */
void oracle_csr_spmm_f64(int64_t M, int64_t K, int64_t N, const int64_t* rp, const int32_t* ci,
                         const float* vals, const float* B, const int64_t* rows, int64_t nrows,
                         double* C, double* S) {
  (void)K;
  int64_t n_out = rows ? nrows : M;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t t = 0; t < n_out; ++t) {
    int64_t i = rows ? rows[t] : t;
    double* c = C + t * N;
    double* s = S ? S + t * N : NULL;
    for (int64_t j = 0; j < N; ++j) { c[j] = 0.0; if (s) s[j] = 0.0; }
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      double a = (double)vals[e];
      const float* b = B + (int64_t)ci[e] * N;
      for (int64_t j = 0; j < N; ++j) c[j] += a * (double)b[j];
      if (s)
        for (int64_t j = 0; j < N; ++j) s[j] += fabs(a) * fabs((double)b[j]);
    }
  }
}

/* Same arithmetic as oracle_csr_spmm_f64, all rows, result rounded to fp32 (the timed CPU
 * baseline: same output bytes as the GPU path). Returns the OpenMP thread count used. */
int oracle_csr_spmm_f32out(int64_t M, int64_t N, const int64_t* rp, const int32_t* ci, const float* vals,
                           const float* B, int64_t row0, int64_t row1, float* C) {
  int nthreads = 1;
#pragma omp parallel
  {
#ifdef _OPENMP
#pragma omp single
    nthreads = omp_get_num_threads();
#endif
    double* acc = (double*)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
#pragma omp for schedule(dynamic, 64)
    for (int64_t i = row0; i < row1; ++i) {
      for (int64_t j = 0; j < N; ++j) acc[j] = 0.0;
      for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
        double a = (double)vals[e];
        const float* b = B + (int64_t)ci[e] * N;
        for (int64_t j = 0; j < N; ++j) acc[j] += a * (double)b[j];
      }
      float* c = C + (i - row0) * N;
      for (int64_t j = 0; j < N; ++j) c[j] = (float)acc[j];
    }
    free(acc);
  }
  (void)M;
  return nthreads;
}

/* ---------------------------------------------------------------- O3: dense brute force */
void oracle_dense_gemm_f64(int64_t M, int64_t K, int64_t N, const double* A, const float* B, double* C) {
  for (int64_t i = 0; i < M; ++i)
    for (int64_t j = 0; j < N; ++j) {
      double s = 0.0;
      for (int64_t k = 0; k < K; ++k) s += A[i * K + k] * (double)B[k * N + j];
      C[i * N + j] = s;
    }
}

/* ---------------------------------------------------------------- O4: CSR -> HRPB */
static int cmp_i32(const void* a, const void* b) {
  int32_t x = *(const int32_t*)a, y = *(const int32_t*)b;
  return (x > y) - (x < y);
}
static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

/* HRPB-v1 byte size of one block with nbr active bricks and nz values (reading R7). */
int64_t oracle_block_bytes(int64_t tk, int64_t nbr, int64_t nz) {
  int64_t hdr = align_up((tk / BRICK_K + 1) + nbr, 8);
  return align_up(hdr + 8 * nbr + 4 * nz, 16);
}

static int check_cfg(int64_t tm, int64_t tk) {
  if (tm <= 0 || tm % BRICK_M || tk <= 0 || tk % BRICK_K) return -1;
  if ((tm / BRICK_M) * (tk / BRICK_K) > 255) return -1;
  return 0;
}

/*
 * Converts panels [p0, p1) of the CSR matrix (panel p = rows [tm*p, min(tm*p+tm, M))).
 * Phase 1: per panel, act = uniq(cols) (sorted ascending, reading R23),
 *   nblk = ceil(nact / tk) (reading R1), blockedRowPtr = exclusive scan.
 * Phase 2: per block: activeCols slice (sentinel K past nact, reading R2),
 *   fill_brick_nnz_pattern, brick-CSC order, row-major values, serialization, sizePtr scan.
 * If the output pointers are NULL only the totals are computed (the "count" pass).
 * Outputs are relative to panel p0: brp[0] = 0, sizePtr[0] = 0.
 * Returns 0, or -1 on a bad configuration.
 */
int oracle_hrpb_convert(int64_t M, int64_t K, const int64_t* rp, const int32_t* ci, const float* vals,
                        int64_t tm, int64_t tk, int64_t p0, int64_t p1,
                        int64_t* num_blocks_out, int64_t* bytes_out,
                        uint32_t* brp, uint32_t* ac, uint64_t* sp, uint8_t* packed) {
  if (check_cfg(tm, tk)) return -1;
  const int64_t nbc = tk / BRICK_K;       /* brick columns per block */
  const int64_t nbrow = tm / BRICK_M;     /* brick rows per block (beta capacity) */
  int64_t nb_total = 0, bytes_total = 0;
  if (brp) brp[0] = 0;
  if (sp) sp[0] = 0;
  /* per-block scratch */
  uint64_t* pat = (uint64_t*)malloc((size_t)(nbrow * nbc) * sizeof(uint64_t));
  float* dense = (float*)malloc((size_t)(tm * tk) * sizeof(float));
  for (int64_t p = p0; p < p1; ++p) {
    int64_t r0 = p * tm, r1 = r0 + tm < M ? r0 + tm : M;
    int64_t e0 = rp[r0], e1 = rp[r1], E = e1 - e0;
    /* Phase 1: act = uniq(cols[row_start : row_end]) */
    int32_t* act = (int32_t*)malloc((size_t)(E > 0 ? E : 1) * sizeof(int32_t));
    memcpy(act, ci + e0, (size_t)E * sizeof(int32_t));
    qsort(act, (size_t)E, sizeof(int32_t), cmp_i32);
    int64_t nact = 0;
    for (int64_t e = 0; e < E; ++e)
      if (nact == 0 || act[nact - 1] != act[e]) act[nact++] = act[e];
    int64_t nblk = (nact + tk - 1) / tk; /* reading R1: ceil */
    /* compacted column id of every entry (ActiveColIdx inverse), and its local row;
     * entries bucketed by block (counting sort) so each block visits only its own entries */
    int64_t* q = (int64_t*)malloc((size_t)(E > 0 ? E : 1) * sizeof(int64_t));
    int64_t* lrow = (int64_t*)malloc((size_t)(E > 0 ? E : 1) * sizeof(int64_t));
    int64_t* bstart = (int64_t*)calloc((size_t)nblk + 1, sizeof(int64_t));
    int64_t* order = (int64_t*)malloc((size_t)(E > 0 ? E : 1) * sizeof(int64_t));
    for (int64_t r = r0; r < r1; ++r)
      for (int64_t e = rp[r]; e < rp[r + 1]; ++e) {
        int32_t* hit = (int32_t*)bsearch(&ci[e], act, (size_t)nact, sizeof(int32_t), cmp_i32);
        q[e - e0] = hit - act;
        lrow[e - e0] = r - r0;
        bstart[q[e - e0] / tk + 1]++;
      }
    for (int64_t j = 0; j < nblk; ++j) bstart[j + 1] += bstart[j];
    {
      int64_t* cur = (int64_t*)malloc((size_t)(nblk > 0 ? nblk : 1) * sizeof(int64_t));
      for (int64_t j = 0; j < nblk; ++j) cur[j] = bstart[j];
      for (int64_t e = 0; e < E; ++e) order[cur[q[e] / tk]++] = e;
      free(cur);
    }
    /* Phase 2: blocks of this panel */
    for (int64_t j = 0; j < nblk; ++j) {
      int64_t b = nb_total + j;
      if (ac)
        for (int64_t t = 0; t < tk; ++t)
          ac[b * tk + t] = (j * tk + t < nact) ? (uint32_t)act[j * tk + t] : (uint32_t)K;
      /* fill_brick_nnz_pattern: dense (tm x tk) view of the block, one bit per stored entry */
      memset(pat, 0, (size_t)(nbrow * nbc) * sizeof(uint64_t));
      memset(dense, 0, (size_t)(tm * tk) * sizeof(float));
      for (int64_t x = bstart[j]; x < bstart[j + 1]; ++x) {
        int64_t e = order[x];
        int64_t lr = lrow[e], lc = q[e] % tk;
        int64_t br = lr / BRICK_M, bc = lc / BRICK_K;
        int64_t bit = (lr % BRICK_M) * BRICK_K + (lc % BRICK_K); /* reading R3 */
        pat[br * nbc + bc] |= (uint64_t)1 << bit;                  /* explicit zeros count: R11 */
        dense[lr * tk + lc] = vals ? vals[e0 + e] : 0.0f;
      }
      /* active bricks in CSC order: brick column ascending, then brick row ascending */
      int64_t nbr = 0, nz = 0;
      for (int64_t bc = 0; bc < nbc; ++bc)
        for (int64_t br = 0; br < nbrow; ++br)
          if (pat[br * nbc + bc]) { ++nbr; nz += __builtin_popcountll(pat[br * nbc + bc]); }
      int64_t size = oracle_block_bytes(tk, nbr, nz);
      if (packed) {
        uint8_t* blk = packed + bytes_total;
        memset(blk, 0, (size_t)size);
        uint8_t* colPtr = blk;
        uint8_t* rows = blk + (nbc + 1);
        int64_t hdr = align_up((nbc + 1) + nbr, 8);
        uint64_t* patterns = (uint64_t*)(blk + hdr);
        float* values = (float*)(blk + hdr + 8 * nbr);
        int64_t k = 0, v = 0;
        colPtr[0] = 0;
        for (int64_t bc = 0; bc < nbc; ++bc) {
          for (int64_t br = 0; br < nbrow; ++br) {
            uint64_t pt = pat[br * nbc + bc];
            if (!pt) continue;
            rows[k] = (uint8_t)br;
            patterns[k] = pt;
            /* values of the brick in row-major (= ascending bit) order (reading R4) */
            for (int bit = 0; bit < 64; ++bit)
              if ((pt >> bit) & 1) {
                int64_t lr = br * BRICK_M + bit / BRICK_K, lc = bc * BRICK_K + bit % BRICK_K;
                values[v++] = dense[lr * tk + lc];
              }
            ++k;
          }
          colPtr[bc + 1] = (uint8_t)k;
        }
      }
      bytes_total += size;
      if (sp) sp[b + 1] = (uint64_t)bytes_total;
    }
    nb_total += nblk;
    if (brp) brp[p - p0 + 1] = (uint32_t)nb_total;
    free(act); free(q); free(lrow); free(bstart); free(order);
  }
  free(pat);
  free(dense);
  if (num_blocks_out) *num_blocks_out = nb_total;
  if (bytes_out) *bytes_out = bytes_total;
  return 0;
}

/* ---------------------------------------------------------------- O5: HRPB -> CSR */
typedef struct { int32_t col; float val; } ent_t;
static int cmp_ent(const void* a, const void* b) {
  int32_t x = ((const ent_t*)a)->col, y = ((const ent_t*)b)->col;
  return (x > y) - (x < y);
}
/* Walks blocks -> bricks -> bits and emits (row, original column, value); rows sorted by
 * column. Returns nnz, or -1 on corrupt metadata / capacity overflow. */
int64_t oracle_hrpb_to_csr(int64_t M, int64_t K, int64_t tm, int64_t tk, const uint32_t* brp, const uint32_t* ac,
                           const uint64_t* sp, const uint8_t* packed, int64_t cap, int64_t* rp_out,
                           int32_t* ci_out, float* v_out) {
  if (check_cfg(tm, tk)) return -1;
  int64_t P = (M + tm - 1) / tm, nbc = tk / BRICK_K, nnz = 0;
  for (int64_t i = 0; i <= M; ++i) rp_out[i] = 0;
  /* pass 1: counts per row */
  for (int pass = 0; pass < 2; ++pass) {
    int64_t* cur = NULL;
    if (pass == 1) {
      for (int64_t i = 0; i < M; ++i) rp_out[i + 1] += rp_out[i];
      nnz = rp_out[M];
      if (nnz > cap) return -1;
      cur = (int64_t*)malloc((size_t)(M > 0 ? M : 1) * sizeof(int64_t));
      for (int64_t i = 0; i < M; ++i) cur[i] = rp_out[i];
    }
    for (int64_t p = 0; p < P; ++p)
      for (uint32_t b = brp[p]; b < brp[p + 1]; ++b) {
        const uint8_t* blk = packed + sp[b];
        const uint8_t* colPtr = blk;
        int64_t nbr = colPtr[nbc];
        const uint8_t* rows = blk + nbc + 1;
        int64_t hdr = align_up((nbc + 1) + nbr, 8);
        const uint64_t* patterns = (const uint64_t*)(blk + hdr);
        const float* values = (const float*)(blk + hdr + 8 * nbr);
        int64_t v = 0;
        for (int64_t bc = 0; bc < nbc; ++bc)
          for (int64_t k = colPtr[bc]; k < colPtr[bc + 1]; ++k) {
            uint64_t pt = patterns[k];
            for (int bit = 0; bit < 64; ++bit)
              if ((pt >> bit) & 1) {
                int64_t row = p * tm + rows[k] * BRICK_M + bit / BRICK_K;
                uint32_t col = ac[(int64_t)b * tk + bc * BRICK_K + bit % BRICK_K];
                if (row >= M || col >= (uint64_t)K) { free(cur); return -1; }
                if (pass == 0) rp_out[row + 1]++;
                else { ci_out[cur[row]] = (int32_t)col; v_out[cur[row]] = values[v]; cur[row]++; }
                ++v;
              }
          }
      }
    if (pass == 1) {
      free(cur);
      for (int64_t i = 0; i < M; ++i) { /* order each row by column */
        int64_t a = rp_out[i], n = rp_out[i + 1] - a;
        ent_t* tmp = (ent_t*)malloc((size_t)(n > 0 ? n : 1) * sizeof(ent_t));
        for (int64_t e = 0; e < n; ++e) { tmp[e].col = ci_out[a + e]; tmp[e].val = v_out[a + e]; }
        qsort(tmp, (size_t)n, sizeof(ent_t), cmp_ent);
        for (int64_t e = 0; e < n; ++e) { ci_out[a + e] = tmp[e].col; v_out[a + e] = tmp[e].val; }
        free(tmp);
      }
    }
  }
  return nnz;
}

/* ---------------------------------------------------------------- O6: invariants */
/* Returns 0 if every invariant holds, else a positive code, message in msg. */
int oracle_hrpb_check(int64_t M, int64_t K, int64_t nnz, int64_t tm, int64_t tk, const uint32_t* brp,
                      const uint32_t* ac, const uint64_t* sp, const uint8_t* packed, char* msg, int msglen) {
#define FAIL(code, ...) do { if (msg) snprintf(msg, (size_t)msglen, __VA_ARGS__); return code; } while (0)
  if (check_cfg(tm, tk)) FAIL(1, "bad config tm=%lld tk=%lld", (long long)tm, (long long)tk);
  int64_t P = (M + tm - 1) / tm, nbc = tk / BRICK_K, nbrow = tm / BRICK_M;
  if (brp[0] != 0) FAIL(2, "blockedRowPtr[0] != 0");
  for (int64_t p = 0; p < P; ++p)
    if (brp[p + 1] < brp[p]) FAIL(3, "blockedRowPtr not monotone at %lld", (long long)p);
  int64_t NB = brp[P];
  if (sp[0] != 0) FAIL(4, "sizePtr[0] != 0");
  int64_t pop = 0;
  for (int64_t b = 0; b < NB; ++b) {
    if (sp[b + 1] <= sp[b]) FAIL(5, "sizePtr not strictly increasing at %lld", (long long)b);
    if ((sp[b + 1] - sp[b]) % 16 || sp[b] % 16) FAIL(6, "block %lld not 16-byte aligned", (long long)b);
  }
  for (int64_t p = 0; p < P; ++p) {
    int64_t r0 = p * tm, nrows = (r0 + tm < M ? tm : M - r0);
    int64_t seen_sentinel = 0;
    int64_t prev = -1;
    for (uint32_t b = brp[p]; b < brp[p + 1]; ++b) {
      for (int64_t t = 0; t < tk; ++t) {
        uint32_t c = ac[(int64_t)b * tk + t];
        if (c == (uint32_t)K) { seen_sentinel = 1; continue; }
        if (seen_sentinel) FAIL(7, "activeCols: real column after sentinel in panel %lld", (long long)p);
        if (c > (uint32_t)K) FAIL(8, "activeCols out of range in block %u", b);
        if ((int64_t)c <= prev) FAIL(9, "activeCols not sorted/unique in panel %lld", (long long)p);
        prev = c;
      }
      if (seen_sentinel && b + 1 < brp[p + 1]) FAIL(10, "sentinel outside the last block of panel %lld", (long long)p);
      const uint8_t* blk = packed + sp[b];
      const uint8_t* colPtr = blk;
      int64_t nbr = colPtr[nbc];
      if (colPtr[0] != 0) FAIL(11, "colPtr[0] != 0 in block %u", b);
      for (int64_t bc = 0; bc < nbc; ++bc)
        if (colPtr[bc + 1] < colPtr[bc]) FAIL(12, "colPtr not monotone in block %u", b);
      const uint8_t* rows = blk + nbc + 1;
      int64_t hdr = align_up((nbc + 1) + nbr, 8);
      const uint64_t* patterns = (const uint64_t*)(blk + hdr);
      int64_t nz = 0;
      for (int64_t bc = 0; bc < nbc; ++bc)
        for (int64_t k = colPtr[bc]; k < colPtr[bc + 1]; ++k) {
          if (rows[k] >= nbrow) FAIL(13, "rows[] out of range in block %u", b);
          if (k > colPtr[bc] && rows[k] <= rows[k - 1]) FAIL(14, "rows not increasing in block %u", b);
          uint64_t pt = patterns[k];
          if (!pt) FAIL(15, "zero pattern stored in block %u", b);
          int full = 1; /* all four columns of the brick are real (non-sentinel) */
          for (int lc = 0; lc < BRICK_K; ++lc) {
            uint32_t c = ac[(int64_t)b * tk + bc * BRICK_K + lc];
            if (c == (uint32_t)K) {
              full = 0;
              for (int lr = 0; lr < BRICK_M; ++lr)
                if ((pt >> (lr * BRICK_K + lc)) & 1) FAIL(16, "bit set in a sentinel column, block %u", b);
            }
          }
          for (int lr = 0; lr < BRICK_M; ++lr) {
            int64_t row = r0 + rows[k] * BRICK_M + lr;
            if (row >= r0 + nrows)
              for (int lc = 0; lc < BRICK_K; ++lc)
                if ((pt >> (lr * BRICK_K + lc)) & 1) FAIL(17, "bit set in a row >= M, block %u", b);
          }
          /* TM == brick_m: every real column has >= 1 nnz in its brick => popcount >= 4 */
          if (tm == BRICK_M && full && __builtin_popcountll(pt) < 4) FAIL(18, "full brick with popcount < 4, block %u", b);
          nz += __builtin_popcountll(pt);
        }
      pop += nz;
      int64_t expect = oracle_block_bytes(tk, nbr, nz);
      if ((int64_t)(sp[b + 1] - sp[b]) != expect) FAIL(19, "block %u size %lld != %lld", b,
                                                          (long long)(sp[b + 1] - sp[b]), (long long)expect);
      /* padding bytes are zero */
      for (int64_t i = (nbc + 1) + nbr; i < hdr; ++i) if (blk[i]) FAIL(20, "nonzero header pad, block %u", b);
      for (int64_t i = hdr + 8 * nbr + 4 * nz; i < expect; ++i) if (blk[i]) FAIL(21, "nonzero tail pad, block %u", b);
    }
    /* the last block of a panel must hold at least one real column */
    if (brp[p + 1] > brp[p] && ac[(int64_t)brp[p + 1] * tk - tk] == (uint32_t)K)
      FAIL(22, "empty block in panel %lld", (long long)p);
  }
  if (pop != nnz) FAIL(23, "sum popcount %lld != nnz %lld", (long long)pop, (long long)nnz);
  return 0;
#undef FAIL
}

/* ---------------------------------------------------------------- O7: HRPB SpMM emulator */
/* Walks HRPB as Alg. "cuTeSpMM kernel design": per panel, per block, gather the TK
 * B rows named by activeCols (sentinel -> zero row), per brick decode the pattern with the
 * prefix count index = popcount(pattern & ((1<<bit)-1)), multiply the zero-filled
 * 16x4 brick with the 4 gathered rows, accumulate; write C once per panel. FP64. */
void oracle_hrpb_spmm_f64(int64_t M, int64_t K, int64_t N, int64_t tm, int64_t tk, const uint32_t* brp,
                          const uint32_t* ac, const uint64_t* sp, const uint8_t* packed, const float* B, double* C) {
  int64_t P = (M + tm - 1) / tm, nbc = tk / BRICK_K;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t p = 0; p < P; ++p) {
    double* acc = (double*)calloc((size_t)(tm * N), sizeof(double));
    for (uint32_t b = brp[p]; b < brp[p + 1]; ++b) {
      const uint8_t* blk = packed + sp[b];
      const uint8_t* colPtr = blk;
      int64_t nbr = colPtr[nbc];
      const uint8_t* rows = blk + nbc + 1;
      int64_t hdr = align_up((nbc + 1) + nbr, 8);
      const uint64_t* patterns = (const uint64_t*)(blk + hdr);
      const float* nnzs = (const float*)(blk + hdr + 8 * nbr);
      int64_t nnz_offset = 0;
      for (int64_t bc = 0; bc < nbc; ++bc)
        for (int64_t j = colPtr[bc]; j < colPtr[bc + 1]; ++j) {
          uint64_t pt = patterns[j];
          double afrag[BRICK_M][BRICK_K];
          for (int bit = 0; bit < 64; ++bit) {
            double a = 0.0;
            if ((pt >> bit) & 1) {
              uint64_t below = bit ? (pt & (((uint64_t)1 << bit) - 1)) : 0;
              a = nnzs[nnz_offset + __builtin_popcountll(below)];
            }
            afrag[bit / BRICK_K][bit % BRICK_K] = a;
          }
          nnz_offset += __builtin_popcountll(pt);
          for (int lr = 0; lr < BRICK_M; ++lr)
            for (int lc = 0; lc < BRICK_K; ++lc) {
              uint32_t col = ac[(int64_t)b * tk + bc * BRICK_K + lc];
              if (col >= (uint64_t)K) continue; /* sentinel row of B is zero */
              double a = afrag[lr][lc];
              double* c = acc + (rows[j] * BRICK_M + lr) * N;
              const float* brow = B + (int64_t)col * N;
              for (int64_t n = 0; n < N; ++n) c[n] += a * (double)brow[n];
            }
        }
    }
    for (int64_t lr = 0; lr < tm && p * tm + lr < M; ++lr)
      memcpy(C + (p * tm + lr) * N, acc + lr * N, (size_t)N * sizeof(double));
    free(acc);
  }
}

/* ---------------------------------------------------------------- O8: row reordering (NEXT-4) */
/* The row permutation of the reordering preprocessing (the paper names matrix reordering as
 * ongoing work, without an algorithm: reading R25 in DESIGN.md). Key of row i:
 *   ((31 - floor(log2(max(deg_i, 1)))) << 40) | min over the row's columns c of h(c),
 *   h(c) = (c * 0x9E3779B97F4A7C15 mod 2^64) >> 40 (24 bits; an empty row: 2^24 - 1),
 * rows sorted by ascending key, ties by ascending row id (a stable sort). perm[i] = the row placed at i. */
typedef struct { uint64_t key; int32_t row; } reo_t;
static int cmp_reo(const void* a, const void* b) {
  const reo_t* x = (const reo_t*)a;
  const reo_t* y = (const reo_t*)b;
  if (x->key != y->key) return x->key < y->key ? -1 : 1;
  return x->row < y->row ? -1 : (x->row > y->row);
}
int oracle_reorder_rows(int64_t M, const int64_t* rp, const int32_t* ci, int32_t* perm) {
  reo_t* r = (reo_t*)malloc((size_t)(M > 0 ? M : 1) * sizeof(reo_t));
  if (!r) return 1;
  for (int64_t i = 0; i < M; ++i) {
    const int64_t deg = rp[i + 1] - rp[i];
    uint64_t lg = 0;
    while (lg < 31 && (2ll << lg) <= deg) ++lg; /* floor(log2(deg)) for deg >= 1, 0 for deg <= 1 */
    uint64_t mh = 0xFFFFFFull;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      const uint64_t h = ((uint64_t)(uint32_t)ci[k] * 0x9E3779B97F4A7C15ull) >> 40;
      if (h < mh) mh = h;
    }
    r[i].key = ((31 - lg) << 40) | mh;
    r[i].row = (int32_t)i;
  }
  qsort(r, (size_t)M, sizeof(reo_t), cmp_reo);
  for (int64_t i = 0; i < M; ++i) perm[i] = r[i].row;
  free(r);
  return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
