"""ctypes binding of libhrpb (include/hrpb.h). Argument marshalling only — every step runs in the
library's sm_100a kernels. Names follow the C ABI: build -> hrpb_build, spmm -> hrpb_spmm, ...
"""
from __future__ import annotations

import ctypes as C
import os
import re

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libhrpb.so")
_HEADER = os.path.join(os.path.dirname(_HERE), "include", "hrpb.h")
_lib = None

STATUS = {0: "HRPB_SUCCESS", 1: "HRPB_ERROR_INVALID_VALUE", 2: "HRPB_ERROR_INVALID_CSR",
          3: "HRPB_ERROR_DIMENSION_MISMATCH", 4: "HRPB_ERROR_OUT_OF_MEMORY", 5: "HRPB_ERROR_NOT_SUPPORTED",
          6: "HRPB_ERROR_CUDA"}


def _header_functions():
    txt = open(_HEADER).read()
    return sorted(set(re.findall(r"^[a-z_0-9 ]+?\**\s*\b(hrpb_[a-z_0-9]+)\(", txt, flags=re.M)))


EXPORTED_SYMBOLS = _header_functions()


class HrpbError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {STATUS.get(status, status)}")


class _Config(C.Structure):
    _fields_ = [("tm", C.c_int32), ("tk", C.c_int32)]  # tm = 0: automatic (hrpb.h)


class _View(C.Structure):
    _fields_ = [("M", C.c_int64), ("K", C.c_int64), ("nnz", C.c_int64), ("num_panels", C.c_int64),
                ("num_blocks", C.c_int64), ("packed_bytes", C.c_int64), ("tm", C.c_int32), ("tk", C.c_int32),
                ("blockedRowPtr", C.c_void_p), ("activeCols", C.c_void_p), ("sizePtr", C.c_void_p),
                ("packedBlocks", C.c_void_p)]


def lib_path() -> str:
    return _SO


def lib():
    """Loads libhrpb.so. Raises if it has not been built — there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(_SO):
            raise ImportError(f"{_SO} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(_SO)
        i64, vp = C.c_int64, C.c_void_p
        L.hrpb_build.argtypes = [i64, i64, i64, vp, vp, vp, C.POINTER(_Config), vp, C.POINTER(vp)]
        L.hrpb_spmm.argtypes = [vp, vp, vp, i64, i64, i64, vp]
        L.hrpb_spmm_sharded.argtypes = [vp, C.POINTER(vp), C.c_int32, i64, vp, i64, i64, i64, vp]
        L.hrpb_reorder_rows.argtypes = [i64, i64, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.hrpb_set_row_map.argtypes = [vp, vp]
        L.hrpb_build_spmm_host.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, vp, C.POINTER(_Config), vp]
        L.hrpb_build_spmm.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, vp, C.POINTER(_Config), vp,
                                      C.POINTER(vp), C.POINTER(C.c_float)]
        L.hrpb_build_spmm_async.argtypes = [i64, i64, i64, i64, vp, vp, vp, vp, vp, C.POINTER(_Config), vp]
        L.hrpb_sync_status.argtypes = [vp, C.POINTER(C.c_float)]
        L.hrpb_free.argtypes = [vp]
        L.hrpb_get_view.argtypes = [vp, C.POINTER(_View)]
        L.hrpb_copy_view_to_host.argtypes = [vp, vp, vp, vp, vp]
        L.hrpb_get_error_string.argtypes = [C.c_int]
        L.hrpb_get_error_string.restype = C.c_char_p
        L.hrpb_last_cuda_error.restype = C.c_int
        L.hrpb_launch_count.restype = C.c_int64
        for f in ("hrpb_build", "hrpb_spmm", "hrpb_spmm_sharded", "hrpb_reorder_rows", "hrpb_set_row_map", "hrpb_build_spmm", "hrpb_build_spmm_async", "hrpb_sync_status",
                  "hrpb_build_spmm_host", "hrpb_free", "hrpb_get_view", "hrpb_copy_view_to_host"):
            getattr(L, f).restype = C.c_int
        _lib = L
    return _lib


def _check(st: int, where: str):
    if st != 0:
        raise HrpbError(st, where)


def _stream(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _dev(t, dtype, name, numel=None, device=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} must have {numel} elements, got {t.numel()}")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, expected {device}")
    return C.c_void_p(t.data_ptr())


def _csr_dev(row_ptr, col_idx, values, M):
    """Device pointers of a CSR (int64 row_ptr [M+1], int32 col_idx [nnz], float32 values [nnz], one device)."""
    import torch
    nnz = int(col_idx.numel()) if hasattr(col_idx, "numel") else -1
    dev = row_ptr.device if hasattr(row_ptr, "device") else None
    return (_dev(row_ptr, torch.int64, "row_ptr", M + 1), _dev(col_idx, torch.int32, "col_idx", None, dev),
            _dev(values, torch.float32, "values", nnz, dev), nnz)


def _out(out, M, N, B):
    """The caller's C buffer: float32, contiguous, (M, N), on B's device — or a new one."""
    import torch
    if out is None:
        return torch.empty((M, N), dtype=torch.float32, device=B.device)
    if tuple(out.shape) != (M, N):
        raise ValueError(f"out must be ({M}, {N}), got {tuple(out.shape)}")
    _dev(out, torch.float32, "out", M * N, B.device)
    return out


def _host(a, dtype, name, shape):
    """Host buffer pointer (numpy array or CPU tensor) with the exact dtype, shape and C-contiguity."""
    import torch
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise TypeError(f"{name} must be a host buffer")
        ok = a.dtype == {np.int64: torch.int64, np.int32: torch.int32, np.float32: torch.float32}[dtype]
        if not ok or tuple(a.shape) != shape or not a.is_contiguous():
            raise TypeError(f"{name} must be a contiguous {np.dtype(dtype).name} buffer of shape {shape}")
        return C.c_void_p(a.data_ptr())
    if not isinstance(a, np.ndarray) or a.dtype != dtype or a.shape != shape or not a.flags.c_contiguous:
        raise TypeError(f"{name} must be a C-contiguous {np.dtype(dtype).name} array of shape {shape}")
    return C.c_void_p(a.ctypes.data)


class Hrpb:
    """Owning wrapper of an hrpb_t handle (immutable HRPB matrix resident in HBM)."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle
        v = _View()
        _check(lib().hrpb_get_view(self._h, C.byref(v)), "hrpb_get_view")
        self.M, self.K, self.nnz = v.M, v.K, v.nnz
        self.num_panels, self.num_blocks, self.packed_bytes = v.num_panels, v.num_blocks, v.packed_bytes
        self.tm, self.tk = v.tm, v.tk
        self._view = v

    @property
    def handle(self):
        return self._h

    def device_pointers(self):
        v = self._view
        return dict(blockedRowPtr=v.blockedRowPtr, activeCols=v.activeCols, sizePtr=v.sizePtr,
                    packedBlocks=v.packedBlocks)

    def to_host(self):
        """(blockedRowPtr u32, activeCols u32, sizePtr u64, packedBlocks u8) as numpy arrays."""
        brp = np.zeros(self.num_panels + 1, np.uint32)
        ac = np.zeros(max(self.num_blocks * self.tk, 1), np.uint32)
        sp = np.zeros(self.num_blocks + 1, np.uint64)
        packed = np.zeros(max(self.packed_bytes, 1), np.uint8)
        _check(lib().hrpb_copy_view_to_host(self._h, brp.ctypes.data, ac.ctypes.data, sp.ctypes.data,
                                            packed.ctypes.data), "hrpb_copy_view_to_host")
        return brp, ac[: self.num_blocks * self.tk], sp, packed[: self.packed_bytes]

    def set_row_map(self, row_map):
        """hrpb_set_row_map (NEXT-4): this handle was built from reordered rows; SpMM writes A row i to C row
        row_map[i] (CUDA int32 tensor [M], kept alive by the handle). None restores the identity."""
        import torch
        ptr = None
        if row_map is not None:
            ptr = _dev(row_map, torch.int32, "row_map", self.M)
        self._row_map = row_map  # (owned by the caller in C; the binding keeps it alive with the handle)
        _check(lib().hrpb_set_row_map(self._h, ptr), "hrpb_set_row_map")

    def free(self):
        if self._h:
            lib().hrpb_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def build(row_ptr, col_idx, values, M: int, K: int, tm: int = 16, tk: int = 16, stream=None) -> Hrpb:
    """hrpb_build: CSR (CUDA tensors int64/int32/float32) -> HRPB handle. tm = 0: the library picks TM."""
    rp, ci, va, nnz = _csr_dev(row_ptr, col_idx, values, M)
    cfg = _Config(tm, tk)
    h = C.c_void_p()
    st = lib().hrpb_build(M, K, nnz, rp, ci, va, C.byref(cfg), _stream(stream), C.byref(h))
    _check(st, "hrpb_build")
    return Hrpb(h)


def spmm(A: Hrpb, B, out=None, stream=None):
    """hrpb_spmm: C = A.B with B a CUDA float32 (K x N) tensor; returns C (M x N)."""
    import torch
    if B.dim() != 2 or B.shape[0] != A.K:
        raise ValueError(f"B must be ({A.K}, N)")
    N = int(B.shape[1])
    out = _out(out, A.M, N, B)
    st = lib().hrpb_spmm(A.handle, _dev(B, torch.float32, "B"), _dev(out, torch.float32, "out"), A.M, A.K, N,
                         _stream(stream))
    _check(st, "hrpb_spmm")
    return out


def spmm_sharded(A: Hrpb, shards, rows_per_shard: int, out=None, stream=None):
    """hrpb_spmm_sharded: C = A.B with B given as row shards: shards[r] is a CUDA float32
    tensor holding B rows [r * rows_per_shard, min((r + 1) * rows_per_shard, K)) — on this device, or another GPU's
    memory mapped here (dist.peer_shards). Returns C (M x N) on the current device."""
    import torch
    shards = list(shards)
    if not shards:
        raise ValueError("at least one shard")
    N = int(shards[0].shape[1]) if shards[0].dim() == 2 else -1
    nsh = len(shards)
    for r, t in enumerate(shards):
        rows = max(0, min((r + 1) * rows_per_shard, A.K) - r * rows_per_shard)
        if t.dim() != 2 or tuple(t.shape) != (rows, N):
            raise ValueError(f"shard {r} must be ({rows}, {N}), got {tuple(t.shape)}")
        if t.dtype != torch.float32 or not t.is_contiguous() or not t.is_cuda:
            raise TypeError(f"shard {r} must be a contiguous CUDA float32 tensor")
    dev = torch.device("cuda", torch.cuda.current_device())
    if out is None:
        out = torch.empty((A.M, N), dtype=torch.float32, device=dev)
    elif tuple(out.shape) != (A.M, N):
        raise ValueError(f"out must be ({A.M}, {N}), got {tuple(out.shape)}")
    else:
        _dev(out, torch.float32, "out", A.M * N)
    ptrs = (C.c_void_p * nsh)(*[t.data_ptr() if t.numel() else 16 for t in shards])  # (empty shard: never read)
    st = lib().hrpb_spmm_sharded(A.handle, ptrs, nsh, int(rows_per_shard), C.c_void_p(out.data_ptr()), A.M, A.K, N,
                                 _stream(stream))
    _check(st, "hrpb_spmm_sharded")
    return out


def reorder_rows(row_ptr, col_idx, values, M: int, K: int, stream=None):
    """hrpb_reorder_rows (NEXT-4): returns (perm, row_ptr_out, col_idx_out, values_out) as CUDA tensors — row i of the
    permuted CSR is input row perm[i]. Build from the permuted CSR, then A.set_row_map(perm)."""
    import torch
    rp, ci, va, nnz = _csr_dev(row_ptr, col_idx, values, M)
    dev = row_ptr.device
    perm = torch.empty(max(M, 1), dtype=torch.int32, device=dev)
    rp2 = torch.empty(M + 1, dtype=torch.int64, device=dev)
    ci2 = torch.empty(max(nnz, 1), dtype=torch.int32, device=dev)
    v2 = torch.empty(max(nnz, 1), dtype=torch.float32, device=dev)
    st = lib().hrpb_reorder_rows(M, K, nnz, rp, ci, va, C.c_void_p(perm.data_ptr()), C.c_void_p(rp2.data_ptr()),
                                 C.c_void_p(ci2.data_ptr()), C.c_void_p(v2.data_ptr()), _stream(stream))
    _check(st, "hrpb_reorder_rows")
    return perm[:M], rp2, ci2[:nnz], v2[:nnz]


def build_spmm(row_ptr, col_idx, values, B, M: int, K: int, out=None, tm: int = 16, tk: int = 16, stream=None,
               keep: bool = False):
    """hrpb_build_spmm: build + SpMM on CUDA tensors in one call (one synchronization). Returns (C, handle or
    None, (build_ms, spmm_ms)) — the phase times are CUDA-event measured on the stream."""
    import torch
    if B.dim() != 2 or B.shape[0] != K:
        raise ValueError(f"B must be ({K}, N)")
    N = int(B.shape[1])
    out = _out(out, M, N, B)
    rp, ci, va, nnz = _csr_dev(row_ptr, col_idx, values, M)
    cfg = _Config(tm, tk)
    h = C.c_void_p()
    ms = (C.c_float * 2)()
    st = lib().hrpb_build_spmm(M, K, N, nnz, rp, ci, va, _dev(B, torch.float32, "B"), _dev(out, torch.float32, "out"),
                               C.byref(cfg), _stream(stream), C.byref(h) if keep else None, ms)
    _check(st, "hrpb_build_spmm")
    return out, (Hrpb(h) if keep else None), (float(ms[0]), float(ms[1]))


def build_spmm_async(row_ptr, col_idx, values, B, M: int, K: int, out, tm: int = 16, tk: int = 16, stream=None):
    """hrpb_build_spmm_async: build + SpMM into `out` without a per-call synchronization once the call is
    graph-replayed; device-detected CSR errors surface at the next sync_status()."""
    import torch
    if B.dim() != 2 or B.shape[0] != K:
        raise ValueError(f"B must be ({K}, N)")
    N = int(B.shape[1])
    out = _out(out, M, N, B)
    rp, ci, va, nnz = _csr_dev(row_ptr, col_idx, values, M)
    cfg = _Config(tm, tk)
    st = lib().hrpb_build_spmm_async(M, K, N, nnz, rp, ci, va, _dev(B, torch.float32, "B"),
                                     _dev(out, torch.float32, "out"), C.byref(cfg), _stream(stream))
    _check(st, "hrpb_build_spmm_async")
    return out


def sync_status(stream=None):
    """hrpb_sync_status: synchronize the stream, raise on an asynchronous INVALID_CSR; returns the (build_ms,
    spmm_ms) phase times of this thread's most recent build_spmm / build_spmm_async call."""
    ms = (C.c_float * 2)()
    st = lib().hrpb_sync_status(_stream(stream), ms)
    _check(st, "hrpb_sync_status")
    return float(ms[0]), float(ms[1])


def build_spmm_host(row_ptr, col_idx, values, B, M: int, K: int, out=None, tm: int = 16, tk: int = 16, stream=None):
    """hrpb_build_spmm_host: the whole hot path from host buffers (numpy or pinned CPU tensors)."""
    N = int(B.shape[1])
    nnz = int(col_idx.shape[0])
    if out is None:
        out = np.empty((M, N), np.float32)
    cfg = _Config(tm, tk)
    st = lib().hrpb_build_spmm_host(M, K, N, nnz, _host(row_ptr, np.int64, "row_ptr", (M + 1,)),
                                    _host(col_idx, np.int32, "col_idx", (nnz,)),
                                    _host(values, np.float32, "values", (nnz,)), _host(B, np.float32, "B", (K, N)),
                                    _host(out, np.float32, "out", (M, N)), C.byref(cfg), _stream(stream))
    _check(st, "hrpb_build_spmm_host")
    return out


def launch_count() -> int:
    return int(lib().hrpb_launch_count())
