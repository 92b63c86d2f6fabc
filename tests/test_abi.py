"""CPU-side checks of the boundary: the C-ABI library loads and exports every symbol include/hrpb.h
declares; the binding refuses to run without CUDA tensors (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2504_06443_b200 as hp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_declares_the_north_star_calls():
    for name in ("hrpb_build", "hrpb_spmm", "hrpb_free"):
        assert name in hp.EXPORTED_SYMBOLS


def test_library_exports_every_header_symbol():
    lib = hp.hrpb.lib()
    for name in hp.EXPORTED_SYMBOLS:
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", hp.lib_path()], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (hrpb_\w+)", out))
    assert set(hp.EXPORTED_SYMBOLS) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", hp.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_sass_uses_tcgen05_and_tma():
    out = subprocess.run(["cuobjdump", "-sass", hp.lib_path()], capture_output=True, text=True).stdout
    assert "UTCHMMA" in out          # tcgen05.mma
    assert "UTMALDG.2D.GATHER4" in out  # TMA tile::gather4
    assert "LDTM" in out             # tcgen05.ld
    assert "HMMA" not in out.replace("UTCHMMA", "")  # no legacy mma.sync path


def test_error_strings_and_null_handling():
    lib = hp.hrpb.lib()
    assert lib.hrpb_get_error_string(2) == b"HRPB_ERROR_INVALID_CSR"
    assert lib.hrpb_free(None) == 0
    out = ctypes.c_void_p()
    # null row_ptr -> INVALID_VALUE before any device work
    assert lib.hrpb_build(4, 4, 0, None, None, None, None, None, ctypes.byref(out)) == 1
    assert out.value is None
    assert lib.hrpb_spmm(None, None, None, 1, 1, 1, None) == 1


def test_binding_rejects_host_tensors():
    import torch
    rp = torch.zeros(5, dtype=torch.int64)
    with pytest.raises(TypeError):
        hp.build(rp, torch.zeros(0, dtype=torch.int32), torch.zeros(0), 4, 4)


def test_unsupported_tile_pairs_rejected_before_device_work():
    lib = hp.hrpb.lib()
    out = ctypes.c_void_p()
    fake = ctypes.c_void_p(16)  # never dereferenced: the (tm, tk) check comes first
    for tm, tk in [(128, 32), (48, 16), (16, 8), (-1, 16), (256, 16)]:
        cfg = hp.hrpb._Config(tm, tk)
        assert lib.hrpb_build(4, 4, 0, fake, None, None, ctypes.byref(cfg), None, ctypes.byref(out)) == 1
        assert lib.hrpb_build_spmm_host(4, 4, 4, 0, fake, None, None, fake, fake, ctypes.byref(cfg), None) == 1
