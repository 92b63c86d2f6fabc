"""Seeded synthetic inputs shared by the oracle and the CUDA path (no method arithmetic here).

The C generators live in ``synth/synth.c`` (compiled to ``synth/libsynth.so``); this module is
the ctypes binding plus the named workload configurations of BASELINE.json.
Every array is produced from a seed by a counter-based hash, so the same call on any machine
returns the same bytes.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "synth.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared",
                               "-o", _SO, src])
    return _SO


class _Csr(C.Structure):
    _fields_ = [("M", C.c_int64), ("K", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("col_idx", C.POINTER(C.c_int32))]


def _L():
    global _lib
    if _lib is None:
        build()
        lib = C.CDLL(_SO)
        i64, u64, f64 = C.c_int64, C.c_uint64, C.c_double
        P = C.POINTER(_Csr)
        lib.synth_banded.argtypes = [i64, i64, i64, i64, u64, P]
        lib.synth_banded_rows.argtypes = [i64, i64, i64, i64, i64, i64, u64, P]
        lib.synth_uniform_d.argtypes = [i64, i64, i64, u64, P]
        lib.synth_bernoulli.argtypes = [i64, i64, f64, u64, P]
        lib.synth_clustered.argtypes = [i64, i64, i64, i64, u64, P]
        lib.synth_fem.argtypes = [i64, i64, i64, u64, P]
        lib.synth_rmat.argtypes = [i64, i64, f64, f64, f64, C.c_int, u64, P]
        for f in ("synth_banded", "synth_banded_rows", "synth_uniform_d", "synth_bernoulli", "synth_clustered", "synth_fem",
                  "synth_rmat"):
            getattr(lib, f).restype = C.c_int
        lib.synth_values_a.argtypes = [i64, i64, C.c_int, u64, C.c_void_p]
        lib.synth_dense.argtypes = [i64, i64, i64, C.c_int, u64, C.c_void_p]
        lib.synth_hash.argtypes = [u64, u64]
        lib.synth_hash.restype = u64
        lib.synth_free.argtypes = [C.c_void_p]
        lib.synth_num_threads.restype = C.c_int
        _lib = lib
    return _lib


def _take(csr: _Csr):
    lib = _L()
    M, nnz = csr.M, csr.nnz
    rp = np.ctypeslib.as_array(csr.row_ptr, shape=(M + 1,)).copy()
    ci = np.ctypeslib.as_array(csr.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
    lib.synth_free(C.cast(csr.row_ptr, C.c_void_p))
    lib.synth_free(C.cast(csr.col_idx, C.c_void_p))
    return rp, ci


def _call(fn, *args):
    o = _Csr()
    rc = fn(*args, C.byref(o))
    if rc != 0:
        raise MemoryError("synth generator failed")
    return _take(o)


def banded(M, K, d=16, w=32, seed=1, r0=0, shift=0):
    """Rows [r0, r0+M) of the banded matrix with K columns (row slabs are independent); row g's
    band is centred at column g - shift."""
    return _call(_L().synth_banded_rows, r0, M, K, d, w, shift, seed)


def uniform_d(M, K, d=8, seed=1):
    return _call(_L().synth_uniform_d, M, K, d, seed)


def bernoulli(M, K, p=0.01, seed=1):
    return _call(_L().synth_bernoulli, M, K, p, seed)


def clustered(M, K, ncl=4, spread=32, seed=1):
    return _call(_L().synth_clustered, M, K, ncl, spread, seed)


def fem(nx=250, ny=250, bs=8, seed=1):
    return _call(_L().synth_fem, nx, ny, bs, seed)


def rmat(scale, ef=32, a=0.57, b=0.19, c=0.19, permute=False, seed=1):
    return _call(_L().synth_rmat, scale, ef, a, b, c, int(permute), seed)


def values_a(nnz, mode, seed=2, e0=0):
    out = np.empty(max(nnz, 0), dtype=np.float32)
    if nnz:
        _L().synth_values_a(e0, nnz, mode, seed, out.ctypes.data)
    return out


def dense(rows, N, mode, seed=3, r0=0):
    out = np.empty((rows, N), dtype=np.float32)
    if rows and N:
        _L().synth_dense(r0, rows, N, mode, seed, out.ctypes.data)
    return out


def splitmix_hash(seed, i):
    return int(_L().synth_hash(seed, i))


def num_threads():
    return int(_L().synth_num_threads())


EXACT, FLOAT = 0, 1


@dataclass
class Workload:
    name: str
    M: int
    K: int
    N: int
    mode: int  # EXACT or FLOAT
    row_ptr: np.ndarray
    col_idx: np.ndarray
    vals: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_idx.shape[0])

    def B(self, seed: int = 3) -> np.ndarray:
        return dense(self.K, self.N, self.mode, seed)


def _w(name, M, K, N, mode, rp, ci):
    return Workload(name, M, K, N, mode, rp, ci, values_a(int(ci.shape[0]), mode, seed=2))


# Named configurations (BASELINE.json "configs").  `scale` shrinks the
# structural size for quick tests while keeping the shape of the distribution.
def make(name: str, N: int | None = None, scale: int = 0, mode: int | None = None) -> Workload:
    s = 1 << scale if scale > 0 else 1
    if name == "c1":  # uniform random 4096^2, 1%, N=32, exact mode
        M = K = 4096 // s
        rp, ci = bernoulli(M, K, 0.01, seed=1)
        return _w(name, M, K, N or 32, EXACT if mode is None else mode, rp, ci)
    if name == "c2a":  # banded 1M^2, 16 distinct cols in [i-32, i+32), N=128, float
        M = K = (1 << 20) // s
        rp, ci = banded(M, K, 16, 32, seed=1)
        return _w(name, M, K, N or 128, FLOAT if mode is None else mode, rp, ci)
    if name == "c2b":  # block-clustered 1M^2, 4 dense 16x4 clusters per panel, N=128, float
        M = K = (1 << 20) // s
        rp, ci = clustered(M, K, 4, 32, seed=1)
        return _w(name, M, K, N or 128, FLOAT if mode is None else mode, rp, ci)
    if name in ("c3", "c3p"):  # R-MAT scale 22, ef 32, N=256, float
        sc = 22 - scale
        rp, ci = rmat(sc, 32, 0.57, 0.19, 0.19, permute=(name == "c3p"), seed=1)
        n = 1 << sc
        return _w(name, n, n, N or 256, FLOAT if mode is None else mode, rp, ci)
    if name == "c4":  # uniform 8 cols/row, 2M^2, N=512, float
        M = K = (1 << 21) // s
        rp, ci = uniform_d(M, K, 8, seed=1)
        return _w(name, M, K, N or 512, FLOAT if mode is None else mode, rp, ci)
    if name == "c5":  # FEM 250x250 nodes x 8 dofs, 8x8 blocks, 9-pt stencil + 1 random, N sweep
        nx = max(2, 250 // s)
        rp, ci = fem(nx, nx, 8, seed=1)
        M = nx * nx * 8
        return _w(name, M, M, N or 128, FLOAT if mode is None else mode, rp, ci)
    raise KeyError(name)


CONFIG_NAMES = ("c1", "c2a", "c2b", "c3", "c3p", "c4", "c5")
