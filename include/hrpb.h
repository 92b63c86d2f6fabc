/*
 * hrpb.h — C ABI of libhrpb: B200-native (sm_100a) HRPB construction and SpMM.
 *
 * Method: cuTeSpMM / HRPB, arxiv 2504.06443 (cited as P:Lnnn = /root/reference/PAPER.md line).
 *   Problem statement (§Notations): C = A.B with A sparse M x K, B dense K x N, C dense M x N.
 *   HRPB (Figs. "Block Data Structure" P:L43-48 and "HRPB data structure" P:L59-64):
 *   rows are grouped into TM-row panels; each panel's active columns are compacted into
 *   (TM, TK) blocks; a block is split into 16 x 4 bricks carrying a 64-bit non-zero pattern and
 *   packed values in brick-CSC order.
 *   Kernel (Alg. "cuTeSpMM kernel design"): per block, gather the TK rows of B named by
 *   activeCols, decode bricks into zero-filled tiles and multiply them on tensor cores.
 *
 * All matrix pointers are DEVICE pointers except in hrpb_build_spmm_host (HOST pointers).
 * Streams are CUDA runtime streams (cudaStream_t); NULL means the legacy default stream.
 * No function aborts or throws; every failure is reported as an hrpb_status_t.
 */
#ifndef HRPB_H_
#define HRPB_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

struct CUstream_st;
typedef struct CUstream_st* hrpb_stream_t; /* == cudaStream_t */

typedef enum {
  HRPB_SUCCESS = 0,
  HRPB_ERROR_INVALID_VALUE = 1,       /* null pointer, negative size, unsupported tm/tk, M or K >= 2^31 */
  HRPB_ERROR_INVALID_CSR = 2,         /* row_ptr not monotone / row_ptr[0] != 0 / row_ptr[M] != nnz /
                                         column out of range / columns not strictly increasing in a row */
  HRPB_ERROR_DIMENSION_MISMATCH = 3,  /* hrpb_spmm M or K differ from the handle's */
  HRPB_ERROR_OUT_OF_MEMORY = 4,
  HRPB_ERROR_NOT_SUPPORTED = 5,       /* current device is not sm_100 (B200) */
  HRPB_ERROR_CUDA = 6                 /* any other CUDA error (see hrpb_last_cuda_error) */
} hrpb_status_t;

/* Tile parameters ("TM either 16 or 32", "TK is set to 16"). The hot path is
 * tm = 16, tk = 16. NULL config => {16, 16}.
 * Supported (tm, tk): tm in {16, 32, 64, 128} with tk = 16; tm in {16, 32, 64} with tk = 32 (NEXT-1: taller panels
 * share gathered B rows between more output rows). Anything else => HRPB_ERROR_INVALID_VALUE, in every
 * entry point, before any work.
 * tm = 0 (automatic): the library samples the CSR on the device (one small kernel and one stream synchronization)
 * and picks tm in {16, 64} from the blocks a sample of 64-row groups forms at each height (DESIGN.md NEXT-1). In
 * hrpb_build_spmm / _async the choice is made on the first call of an argument set and kept for its replays. */
typedef struct {
  int32_t tm; /* rows per panel: 16 (0 = automatic) */
  int32_t tk; /* compacted columns per block: 16 */
} hrpb_config_t;

typedef struct hrpb_handle* hrpb_t;

/* Device view of a built HRPB (HRPB-v1 layout, reading R7). Pointers are owned by the
 * handle and valid until hrpb_free. Block b occupies packedBlocks[sizePtr[b] .. sizePtr[b+1]):
 *   u8 colPtr[tk/4+1] | u8 rows[nbr] | zero pad to 8 | u64 patterns[nbr] | f32 values[nz] | pad 16. */
typedef struct {
  int64_t M, K, nnz;
  int64_t num_panels;   /* ceil(M / tm) */
  int64_t num_blocks;   /* NUM_BLKS */
  int64_t packed_bytes; /* sizePtr[num_blocks] */
  int32_t tm, tk;
  const uint32_t* blockedRowPtr; /* [num_panels + 1], first block of each panel */
  const uint32_t* activeCols;    /* [num_blocks * tk], original column id; K = padding (R2) */
  const uint64_t* sizePtr;       /* [num_blocks + 1], byte offset of each block (R8) */
  const uint8_t* packedBlocks;   /* [packed_bytes] */
} hrpb_view_t;

/*
 * hrpb_build — CSR -> HRPB on the GPU (steps B1..B5 of SURVEY §8(a); P:L81-149 Phase 1/2).
 *   M, K, nnz : dimensions of A (0 allowed); M, K < 2^31.
 *   row_ptr   : device int64 [M+1], row_ptr[0] = 0, non-decreasing, row_ptr[M] = nnz.
 *   col_idx   : device int32 [nnz], 0 <= col < K, strictly increasing within a row.
 *   values    : device float [nnz] (bits copied verbatim; explicit zeros are structural, R11).
 *   cfg       : NULL ({16, 16}) or a supported (tm, tk) pair, tm = 0 for the automatic choice (see hrpb_config_t).
 *   stream    : all work is enqueued on it; the call synchronizes it once at the end to read
 *               back sizes and the validation status, so the CSR buffers may be freed on return.
 *   out       : receives the handle (set to NULL on any error).
 * The result is bit-identical to the CPU oracle converter for the same CSR.
 * Errors: INVALID_VALUE, INVALID_CSR, OUT_OF_MEMORY, NOT_SUPPORTED, CUDA.
 */
hrpb_status_t hrpb_build(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                         const float* values, const hrpb_config_t* cfg, hrpb_stream_t stream, hrpb_t* out);

/*
 * hrpb_spmm — C = A.B (Alg. "cuTeSpMM kernel design" P:L170-231), steps S1..S5.
 *   A : handle from hrpb_build (immutable; concurrent calls on different streams are allowed
 *       when each call has its own C).
 *   B : device float, row-major K x N (ld = N), finite values (R17). Must not alias C.
 *   C : device float, row-major M x N (ld = N); fully overwritten (empty rows become 0, R13).
 *   M, K must equal the handle's (else DIMENSION_MISMATCH); N >= 0 (N = 0 is a no-op).
 * Arithmetic: TF32 tensor cores (A rounded to nearest TF32, ties away — cvt.rna semantics, done with integer ops;
 * B truncated by the tensor core), FP32 accumulation in TMEM. A must be finite too (a NaN payload may round to Inf).
 * Work split (S1): one persistent CTA per SM takes a contiguous range of equal cost (1 per block + w per panel
 * epilogue, w = 5 / 5 / 12 / 24 at TM = 16 / 32 / 64 / 128, DESIGN.md NEXT-2); on long launches (nnz >= 64M,
 * TM <= 32) the work is cut into 16 guided shares per SM that the CTAs claim dynamically. A panel larger than two
 * shares is split between them: partial tiles go to a per-call workspace and a fix-up kernel adds them in share
 * order. Within a panel the blocks alternate between two TMEM accumulator sets that the epilogue adds. Results are
 * deterministic for a given (handle, N) and launch configuration, but the bits of a split panel's rows may differ
 * between configurations (e.g. the chunked launches of hrpb_build_spmm_host).
 * Scratch (the split-panel workspace, a padded copy of B when its rows are not 16-B aligned) is allocated per
 * call, stream-ordered (so concurrent calls on different streams never share it). Asynchronous on `stream`; no
 * host synchronization. A call on a stream other than the build stream is recorded on the handle so that
 * hrpb_free orders the release after it.
 */
hrpb_status_t hrpb_spmm(const hrpb_t A, const float* B, float* C, int64_t M, int64_t K, int64_t N,
                        hrpb_stream_t stream);

/*
 * hrpb_spmm_sharded — C = A.B with B ROW-SHARDED (the repeated-SpMM use case of P:L484 with a
 * B too large or too costly to replicate): shard r holds B rows [r*rows_per_shard, min((r+1)*rows_per_shard, K))
 * as a row-major (rows x N) array, ld = N. Each gathered B row (S3) is read from its shard in place: a shard may be
 * local device memory or another GPU's memory mapped into this device's address space (CUDA IPC / peer access
 * over NVLink), so no B replica and no broadcast are needed. Same kernel, arithmetic, determinism and work split
 * as hrpb_spmm (the result is bit-identical to hrpb_spmm on the concatenated B).
 *   shards         : HOST array [nshards] of device pointers, each 16-B aligned; read-only, owned by the caller,
 *                    valid until the call's work on `stream` has completed.
 *   nshards        : 1..32 and equal to ceil(K / rows_per_shard) (1 when K = 0).
 *   rows_per_shard : >= 1.
 *   N              : >= 0 and a multiple of 4 (rows stay 16-B aligned: no padded copy is made).
 *   C, M, K, stream: as for hrpb_spmm.
 * Errors: INVALID_VALUE (shard table, alignment or N), DIMENSION_MISMATCH, NOT_SUPPORTED, OUT_OF_MEMORY, CUDA.
 */
hrpb_status_t hrpb_spmm_sharded(const hrpb_t A, const float* const* shards, int32_t nshards, int64_t rows_per_shard,
                                float* C, int64_t M, int64_t K, int64_t N, hrpb_stream_t stream);

/*
 * hrpb_reorder_rows — NEXT-4 (the paper's "Matrix Reordering"): a row permutation that puts
 * rows with overlapping column sets into the same TM-row panel (fewer distinct columns per panel, fewer blocks,
 * denser bricks), computed on the GPU, and the row-permuted CSR. Key of row i, sorted ascending and stably:
 * (31 - floor(log2(max(deg_i, 1)))) << 40 | min over the row's columns c of ((c * 0x9E3779B97F4A7C15) mod 2^64) >> 40
 * (degree buckets largest first, then the min-hash of the column set; empty rows: min-hash 2^24 - 1).
 *   M, K, nnz, row_ptr, col_idx, values : the input CSR (device, as for hrpb_build; assumed valid — row pointers are
 *                                         clamped into [0, nnz] so an invalid one cannot read out of bounds).
 *   perm        : device int32 [M], out: row i of the output is row perm[i] of the input.
 *   row_ptr_out : device int64 [M + 1], col_idx_out : device int32 [nnz], values_out : device float [nnz], out: the
 *                 permuted CSR (entries of each row in their original order). Caller-owned, not aliasing the input.
 * Build the HRPB from the permuted CSR, then hrpb_set_row_map(A, perm): hrpb_spmm then writes C in the ORIGINAL
 * row order. Synchronizes nothing (async on `stream`).
 * Errors: INVALID_VALUE, OUT_OF_MEMORY, CUDA.
 */
hrpb_status_t hrpb_reorder_rows(int64_t M, int64_t K, int64_t nnz, const int64_t* row_ptr, const int32_t* col_idx,
                                const float* values, int32_t* perm, int64_t* row_ptr_out, int32_t* col_idx_out,
                                float* values_out, hrpb_stream_t stream);

/*
 * hrpb_set_row_map — declares that A was built from row-permuted rows: hrpb_spmm / hrpb_spmm_sharded write A's row i
 * into C row row_map[i] (device int32 [M], a permutation of 0..M-1, caller-owned, valid while the handle is used;
 * NULL restores the identity). Supported with TK = 16 and the default cp.async gather (hrpb_spmm); other
 * configurations and hrpb_spmm_sharded then return NOT_SUPPORTED. Errors: INVALID_VALUE (A NULL).
 */
hrpb_status_t hrpb_set_row_map(hrpb_t A, const int32_t* row_map);

/*
 * hrpb_build_spmm — the whole hot path on device buffers in one call: hrpb_build then hrpb_spmm, enqueued
 * back to back on `stream` (the SpMM does not wait for the build's size read-back), one synchronization at the
 * end. Arguments as for hrpb_build / hrpb_spmm (all DEVICE pointers).
 *   out      : NULL (the handle is released) or receives the handle (NULL on error).
 *   phase_ms : NULL or float[2] receiving the build and SpMM phase times measured with CUDA events on `stream`.
 * Errors as hrpb_build / hrpb_spmm; an INVALID_CSR input is reported after the SpMM ran, C is then undefined.
 * Replay: when the same arguments (pointers, sizes, config, stream, device) come twice in a row with out == NULL,
 * the second call captures the whole enqueue sequence (allocations, kernels, read-back, frees) into a CUDA graph
 * and later identical calls launch that graph (one host call, no launch gaps between the dependent kernels).
 * Requires a non-default stream (capture is not possible on the legacy default stream: those calls stay eager).
 * HRPB_NO_GRAPH=1 disables it.
 */
hrpb_status_t hrpb_build_spmm(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr,
                              const int32_t* col_idx, const float* values, const float* B, float* C,
                              const hrpb_config_t* cfg, hrpb_stream_t stream, hrpb_t* out, float* phase_ms);

/*
 * hrpb_build_spmm_async — hrpb_build_spmm without the per-call synchronization, for streams of repeated calls
 * (the serving loop, the bench's timed steps). Same arguments as hrpb_build_spmm with out == NULL and no phase
 * times. Once the call has been replayed as a CUDA graph (from the second identical call on, see above) it only
 * launches the graph and returns: CSR errors the device detects (INVALID_CSR) are then reported by the next
 * hrpb_sync_status on that stream, which returns the OR of every such replay since its previous call — as CUDA
 * reports asynchronous kernel faults at a later synchronizing call. Until then, and whenever the arguments
 * change, it behaves exactly like hrpb_build_spmm (synchronous, status returned directly). Argument checks
 * (INVALID_VALUE, NOT_SUPPORTED) are always synchronous. C is valid after the stream is synchronized.
 */
hrpb_status_t hrpb_build_spmm_async(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr,
                                    const int32_t* col_idx, const float* values, const float* B, float* C,
                                    const hrpb_config_t* cfg, hrpb_stream_t stream);

/*
 * hrpb_sync_status — synchronizes `stream`; returns INVALID_CSR if any asynchronous replay since the previous
 * call found an invalid CSR (then clears that state; the state is per device and read-and-cleared in one device
 * atomic, so a replay on another stream can never have its report erased), else HRPB_SUCCESS.
 *   phase_ms : NULL or float[2] receiving the build and SpMM phase times of this thread's most recent
 *              hrpb_build_spmm / hrpb_build_spmm_async call (CUDA events on its stream).
 */
hrpb_status_t hrpb_sync_status(hrpb_stream_t stream, float* phase_ms);

/*
 * hrpb_build_spmm_host — the whole hot path from HOST buffers (end-to-end entry point):
 * H2D copies of the CSR and B, hrpb_build, hrpb_spmm, D2H copy of C, returning after C is in host memory.
 * Pipelined: the CSR and then B (in 32 row chunks) are copied on a library-owned copy stream, the build runs on
 * `stream` once the CSR is in, C is computed in 16 panel chunks — each starting as soon as the B rows up to its
 * largest active column have arrived — and each chunk is copied back on a second library stream while later B
 * chunks are still in flight. Host buffers should be pinned for full (and overlapped) PCIe bandwidth.
 * Arguments as for hrpb_build / hrpb_spmm, with host pointers.
 */
hrpb_status_t hrpb_build_spmm_host(int64_t M, int64_t K, int64_t N, int64_t nnz, const int64_t* row_ptr_h,
                                   const int32_t* col_idx_h, const float* values_h, const float* B_h, float* C_h,
                                   const hrpb_config_t* cfg, hrpb_stream_t stream);

/* Releases the handle's device memory, stream-ordered on the build stream after every hrpb_spmm recorded on
 * other streams (event waits; more than 8 distinct streams: a device synchronization). Returns without waiting.
 * NULL is a no-op. */
hrpb_status_t hrpb_free(hrpb_t A);

/* Fills *view with the handle's metadata and device pointers. */
hrpb_status_t hrpb_get_view(const hrpb_t A, hrpb_view_t* view);

/* Test/introspection: copies the four HRPB arrays to HOST buffers sized from hrpb_get_view
 * (blockedRowPtr [num_panels+1] u32, activeCols [num_blocks*tk] u32, sizePtr [num_blocks+1] u64,
 * packedBlocks [packed_bytes] u8). Any destination may be NULL to skip it. Synchronous. */
hrpb_status_t hrpb_copy_view_to_host(const hrpb_t A, uint32_t* blockedRowPtr, uint32_t* activeCols, uint64_t* sizePtr,
                                     uint8_t* packedBlocks);

/* Human-readable name of a status code (static storage). */
const char* hrpb_get_error_string(hrpb_status_t status);

/* cudaError_t value behind the last HRPB_ERROR_CUDA on this thread (0 if none). */
int hrpb_last_cuda_error(void);

/* Number of kernel launches the library enqueued since process start (instrumentation for the
 * bench's gpu_launches count). */
int64_t hrpb_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HRPB_H_ */
