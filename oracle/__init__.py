"""CPU oracle for HRPB SpMM — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package. The product path (``paper_2504_06443_b200``)
never imports it and shares no code with ``oracle/oracle.c``.

Functions follow /root/reference/PAPER.md (cited as P:Lnnn) step by step; see oracle.c for the
per-function citations and DESIGN.md for the readings (R1..R24) where the paper is silent.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

BRICK_M, BRICK_K = 16, 4


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, src])
    return _SO


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def _L():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_SO)
        i64, vp = C.c_int64, C.c_void_p
        lib.oracle_csr_validate.argtypes = [i64, i64, i64, vp, vp]
        lib.oracle_csr_validate.restype = C.c_int
        lib.oracle_csr_spmm_f64.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, i64, vp, vp]
        lib.oracle_csr_spmm_f32out.argtypes = [i64, i64, vp, vp, vp, vp, i64, i64, vp]
        lib.oracle_csr_spmm_f32out.restype = C.c_int
        lib.oracle_dense_gemm_f64.argtypes = [i64, i64, i64, vp, vp, vp]
        lib.oracle_block_bytes.argtypes = [i64, i64, i64]
        lib.oracle_block_bytes.restype = i64
        lib.oracle_hrpb_convert.argtypes = [i64, i64, vp, vp, vp, i64, i64, i64, i64,
                                            C.POINTER(i64), C.POINTER(i64), vp, vp, vp, vp]
        lib.oracle_hrpb_convert.restype = C.c_int
        lib.oracle_hrpb_to_csr.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, i64, vp, vp, vp]
        lib.oracle_hrpb_to_csr.restype = i64
        lib.oracle_hrpb_check.argtypes = [i64, i64, i64, i64, i64, vp, vp, vp, vp, C.c_char_p, C.c_int]
        lib.oracle_hrpb_check.restype = C.c_int
        lib.oracle_hrpb_spmm_f64.argtypes = [i64, i64, i64, i64, i64, vp, vp, vp, vp, vp, vp]
        lib.oracle_reorder_rows.argtypes = [i64, vp, vp, vp]
        lib.oracle_num_threads.restype = C.c_int
        _lib = lib
    return _lib


def _c(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


# ------------------------------------------------------------------ O1
def csr_validate(M, K, row_ptr, col_idx) -> int:
    rp, ci = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    return int(_L().oracle_csr_validate(M, K, ci.shape[0], _p(rp), _p(ci)))


# ------------------------------------------------------------------ O2
def csr_spmm(M, K, row_ptr, col_idx, vals, B, rows=None, with_bound=False):
    """C = A.B in FP64. Returns C (and S = sum |a||b| if with_bound) for `rows`."""
    rp, ci, v = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(vals, np.float32)
    Bc = _c(B, np.float32)
    N = Bc.shape[1]
    r = None if rows is None else _c(rows, np.int64)
    n_out = M if r is None else r.shape[0]
    Cm = np.empty((n_out, N), dtype=np.float64)
    Sm = np.empty((n_out, N), dtype=np.float64) if with_bound else None
    _L().oracle_csr_spmm_f64(M, K, N, _p(rp), _p(ci), _p(v), _p(Bc), _p(r), n_out, _p(Cm), _p(Sm))
    return (Cm, Sm) if with_bound else Cm


def csr_spmm_f32out(M, row_ptr, col_idx, vals, B, row0=0, row1=None, out=None):
    """Timed CPU baseline: same FP64 arithmetic, fp32 result. Returns (C, threads)."""
    rp, ci, v = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(vals, np.float32)
    Bc = _c(B, np.float32)
    N = Bc.shape[1]
    row1 = M if row1 is None else row1
    Cm = out if out is not None else np.empty((row1 - row0, N), dtype=np.float32)
    th = _L().oracle_csr_spmm_f32out(M, N, _p(rp), _p(ci), _p(v), _p(Bc), row0, row1, _p(Cm))
    return Cm, int(th)


# ------------------------------------------------------------------ O3
def dense_gemm(A_dense, B):
    A = _c(A_dense, np.float64)
    Bc = _c(B, np.float32)
    M, K = A.shape
    N = Bc.shape[1]
    Cm = np.empty((M, N), dtype=np.float64)
    _L().oracle_dense_gemm_f64(M, K, N, _p(A), _p(Bc), _p(Cm))
    return Cm


# ------------------------------------------------------------------ O4
def block_bytes(tk, nbr, nz):
    return int(_L().oracle_block_bytes(tk, nbr, nz))


class Hrpb:
    """Host HRPB arrays produced by the oracle converter (HRPB-v1 byte layout)."""

    def __init__(self, M, K, tm, tk, brp, ac, sp, packed):
        self.M, self.K, self.tm, self.tk = M, K, tm, tk
        self.blockedRowPtr, self.activeCols, self.sizePtr, self.packedBlocks = brp, ac, sp, packed

    @property
    def num_blocks(self):
        return int(self.sizePtr.shape[0] - 1)


def csr_to_hrpb(M, K, row_ptr, col_idx, vals, tm=16, tk=16, p0=0, p1=None) -> Hrpb:
    """CSR -> HRPB for panels [p0, p1). Arrays relative to panel p0."""
    rp, ci, v = _c(row_ptr, np.int64), _c(col_idx, np.int32), _c(vals, np.float32)
    P = (M + tm - 1) // tm
    p1 = P if p1 is None else p1
    nb, nbytes = C.c_int64(0), C.c_int64(0)
    lib = _L()
    rc = lib.oracle_hrpb_convert(M, K, _p(rp), _p(ci), _p(v), tm, tk, p0, p1, C.byref(nb), C.byref(nbytes),
                                 None, None, None, None)
    if rc != 0:
        raise ValueError("oracle_hrpb_convert: bad configuration")
    brp = np.zeros(p1 - p0 + 1, dtype=np.uint32)
    ac = np.zeros(max(nb.value, 0) * tk, dtype=np.uint32)
    sp = np.zeros(nb.value + 1, dtype=np.uint64)
    packed = np.zeros(max(nbytes.value, 1), dtype=np.uint8)
    lib.oracle_hrpb_convert(M, K, _p(rp), _p(ci), _p(v), tm, tk, p0, p1, None, None,
                            _p(brp), _p(ac), _p(sp), _p(packed))
    return Hrpb(M, K, tm, tk, brp, ac, sp, packed[: nbytes.value])


# ------------------------------------------------------------------ O5
def hrpb_to_csr(h: Hrpb, cap: int):
    rp = np.zeros(h.M + 1, dtype=np.int64)
    ci = np.zeros(max(cap, 1), dtype=np.int32)
    v = np.zeros(max(cap, 1), dtype=np.float32)
    packed = h.packedBlocks if h.packedBlocks.size else np.zeros(1, np.uint8)
    nnz = _L().oracle_hrpb_to_csr(h.M, h.K, h.tm, h.tk, _p(h.blockedRowPtr), _p(h.activeCols), _p(h.sizePtr),
                                  _p(packed), cap, _p(rp), _p(ci), _p(v))
    if nnz < 0:
        raise ValueError("oracle_hrpb_to_csr: corrupt HRPB")
    return rp, ci[:nnz], v[:nnz]


# ------------------------------------------------------------------ O6
def hrpb_check(h: Hrpb, nnz: int):
    """Returns (code, message); code 0 means every invariant holds."""
    buf = C.create_string_buffer(256)
    packed = h.packedBlocks if h.packedBlocks.size else np.zeros(1, np.uint8)
    ac = h.activeCols if h.activeCols.size else np.zeros(1, np.uint32)
    code = _L().oracle_hrpb_check(h.M, h.K, nnz, h.tm, h.tk, _p(h.blockedRowPtr), _p(ac), _p(h.sizePtr),
                                  _p(packed), buf, 256)
    return int(code), buf.value.decode()


# ------------------------------------------------------------------ O7
def hrpb_spmm(h: Hrpb, B):
    Bc = _c(B, np.float32)
    N = Bc.shape[1]
    Cm = np.zeros((h.M, N), dtype=np.float64)
    packed = h.packedBlocks if h.packedBlocks.size else np.zeros(1, np.uint8)
    ac = h.activeCols if h.activeCols.size else np.zeros(1, np.uint32)
    _L().oracle_hrpb_spmm_f64(h.M, h.K, N, h.tm, h.tk, _p(h.blockedRowPtr), _p(ac), _p(h.sizePtr),
                              _p(packed), _p(Bc), _p(Cm))
    return Cm


def reorder_rows(M, row_ptr, col_idx):
    """O8: the NEXT-4 row permutation (degree buckets descending, then the column-set min-hash; stable)."""
    rp, ci = _c(row_ptr, np.int64), _c(col_idx, np.int32)
    perm = np.zeros(max(M, 1), np.int32)
    if _L().oracle_reorder_rows(M, _p(rp), _p(ci), _p(perm)) != 0:
        raise MemoryError("oracle_reorder_rows")
    return perm[:M]


def num_threads():
    return int(_L().oracle_num_threads())


def densify(M, K, row_ptr, col_idx, vals):
    A = np.zeros((M, K), dtype=np.float64)
    for i in range(M):
        for e in range(int(row_ptr[i]), int(row_ptr[i + 1])):
            A[i, int(col_idx[e])] = float(vals[e])
    return A
