"""B200-native (sm_100a) HRPB SpMM — the hot path of cuTeSpMM (arxiv 2504.06443).

The compute path is the C-ABI library ``libhrpb.so`` (include/hrpb.h, sources in csrc/):
GPU CSR->HRPB builder kernels and a tcgen05/TMA SpMM kernel. This package is a thin ctypes
binding (argument marshalling only); torch supplies device memory, streams and process groups.
There is no CPU fallback: if the extension is missing or the device is not sm_100, calls raise.
"""
from .hrpb import (Hrpb, HrpbError, build, spmm, spmm_sharded, reorder_rows, build_spmm, build_spmm_async, sync_status, build_spmm_host, launch_count, lib_path,  # noqa: F401
                   EXPORTED_SYMBOLS)
