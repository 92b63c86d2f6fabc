"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on the same seeded inputs.

HRPB construction: byte-identical arrays (blockedRowPtr, activeCols, sizePtr, packedBlocks).
SpMM exact mode: bit-identical C. Float mode: |C - C_ref| <= 4*2^-11*sum|a||b| + 1e-6 (north star).
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import check_exact, check_float, rand_csr

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2504_06443_b200 as hp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def gpu_build(M, K, rp, ci, v, tm=16, tk=16):
    return hp.build(dev(rp), dev(ci), dev(v), M, K, tm=tm, tk=tk)


def assert_same_hrpb(A, ref, what=""):
    brp, ac, sp, packed = A.to_host()
    assert np.array_equal(brp, ref.blockedRowPtr), f"{what}: blockedRowPtr"
    assert np.array_equal(ac, ref.activeCols), f"{what}: activeCols"
    assert np.array_equal(sp, ref.sizePtr), f"{what}: sizePtr"
    assert packed.tobytes() == ref.packedBlocks.tobytes(), f"{what}: packedBlocks"


# --------------------------------------------------------------------------- builder (B1..B5)
BUILD_CASES = [("c1", 0), ("c2a", 5), ("c2b", 5), ("c3", 8), ("c3p", 8), ("c4", 6), ("c5", 3)]


@pytest.mark.parametrize("name,scale", BUILD_CASES)
def test_builder_bit_exact_configs(name, scale):
    w = synth.make(name, scale=scale)
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    ref = oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    assert A.num_blocks == ref.num_blocks
    assert_same_hrpb(A, ref, name)
    assert oracle.hrpb_check(ref, w.nnz)[0] == 0


@pytest.mark.parametrize("seed", range(8))
def test_builder_bit_exact_random_ragged(seed):
    rng = np.random.default_rng(seed)
    M, K = int(rng.integers(1, 400)), int(rng.integers(1, 3000))
    rp, ci, v = rand_csr(M, K, float(rng.choice([0.001, 0.01, 0.1, 0.5])), seed, exact=False)
    A = gpu_build(M, K, rp, ci, v)
    assert_same_hrpb(A, oracle.csr_to_hrpb(M, K, rp, ci, v), f"seed {seed}")


def test_builder_edge_cases():
    # empty matrix, single nnz, K = 1, explicit zeros, dense panel, a hub panel (> 2048 entries)
    cases = []
    cases.append((40, 30, np.zeros(41, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32)))
    cases.append((17, 9, np.array([0] * 17 + [1], np.int64), np.array([8], np.int32), np.array([3.5], np.float32)))
    rp = np.arange(34, dtype=np.int64); rp[-1] = 33
    cases.append((33, 1, np.arange(34, dtype=np.int64), np.zeros(33, np.int32), np.zeros(33, np.float32)))
    d = np.ones((16, 64), bool)
    cases.append((16, 64, np.arange(0, 16 * 64 + 1, 64, dtype=np.int64), np.tile(np.arange(64, dtype=np.int32), 16),
                  np.arange(16 * 64, dtype=np.float32)))
    rng = np.random.default_rng(0)
    hub_cols = [np.sort(rng.choice(100000, 3000, replace=False)).astype(np.int32) for _ in range(20)]
    rp = np.zeros(21, np.int64); rp[1:] = np.cumsum([len(c) for c in hub_cols])
    cases.append((20, 100000, rp, np.concatenate(hub_cols), rng.random(int(rp[-1])).astype(np.float32)))
    for i, (M, K, rp, ci, v) in enumerate(cases):
        A = gpu_build(M, K, rp, ci, v)
        assert_same_hrpb(A, oracle.csr_to_hrpb(M, K, rp, ci, v), f"edge case {i}")


@pytest.mark.parametrize("name", ["c5", "c2a", "c2b", "c3"])
@pytest.mark.parametrize("tm,tk", [(32, 16), (64, 16), (16, 32), (128, 16)])
def test_builder_other_tiles(tm, tk, name):
    w = synth.make(name, scale={"c5": 4, "c2a": 5, "c2b": 5, "c3": 8}[name])
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm, tk=tk)
    assert_same_hrpb(A, oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm, tk=tk), f"{tm}x{tk}")


@pytest.mark.parametrize("tm", [16, 64])
def test_builder_span_boundaries(tm):
    # warp-path ranking variants by panel column span: byte map (span < 768), bitmap atomics (< 8192), warp sort
    # (wider, <= 256 entries) and the listed CTA path; spans straddle each boundary, panels start at random offsets
    rng = np.random.default_rng(tm)
    spans = [1, 31, 32, 33, 700, 767, 768, 769, 800, 4000, 8191, 8192, 8193, 50000]
    K = 60000
    rows, cols = [], []
    for span in spans:
        for _ in range(3):
            base = int(rng.integers(0, K - span + 1))
            for r in range(tm):
                k = int(rng.integers(1, min(span, 12) + 1))
                c = np.sort(rng.choice(span, k, replace=False)) + base
                if r == 0:
                    c = np.unique(np.concatenate([c, [base, base + span - 1]]))
                cols.append(c.astype(np.int32))
    M = len(cols)
    rp = np.zeros(M + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols)
    v = rng.standard_normal(ci.size).astype(np.float32)
    A = gpu_build(M, K, rp, ci, v, tm=tm)
    assert_same_hrpb(A, oracle.csr_to_hrpb(M, K, rp, ci, v, tm=tm), f"spans tm={tm}")


@pytest.mark.parametrize("K,tm", [(10 ** 6 + 7, 16), (10 ** 6 + 7, 64), (10 ** 6 + 7, 128), (2 ** 22 + 3, 16),
                                  (2 ** 23, 32), (2 ** 23 + 5, 16)])
def test_builder_listed_and_hub_paths(K, tm):
    # scattered (R-MAT-like) panels of every listed size class: CTA path (<= 2048 entries: windowed, two-level
    # word bitmap for K <= 2^22, else radix sort) and hub panels (two-level bitmap for K <= 2^23 with staged /
    # streamed entries, masks in shared / global memory, brick patterns in the window / by global atomics;
    # dense column passes above 2^23); panel sizes straddle the class boundaries
    rng = np.random.default_rng(K % 1000 + tm)
    per_row_total = [300, 2047, 2049, 8000, 8300, 20000, 40000]
    cols = []
    for tot in per_row_total:
        for r in range(tm):
            k = max(1, tot // tm + int(rng.integers(-2, 3)))
            lo = 0 if r % 3 else K // 2  # hub-like rows next to rows confined to the upper half
            c = np.sort(rng.choice(K - lo, min(k, K - lo), replace=False)) + lo
            cols.append(c.astype(np.int32))
    M = len(cols) + 5  # ragged tail: 5 empty rows
    cols += [np.zeros(0, np.int32)] * 5
    rp = np.zeros(M + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols)
    v = rng.standard_normal(ci.size).astype(np.float32)
    A = gpu_build(M, K, rp, ci, v, tm=tm)
    assert_same_hrpb(A, oracle.csr_to_hrpb(M, K, rp, ci, v, tm=tm), f"K={K} tm={tm}")


@pytest.mark.parametrize("E", [4000, 12000])
@pytest.mark.parametrize("defect", ["unsorted", "duplicate", "range"])
def test_builder_hub2_rejects_invalid_csr(E, defect):
    # the two-level hub path with staged (4000) and streamed (12000) entries: every defect is reported
    rng = np.random.default_rng(E)
    K = 3 * 10 ** 6
    cols = [np.sort(rng.choice(K, E // 16, replace=False)).astype(np.int32) for _ in range(16)]
    r = cols[9].copy()
    if defect == "unsorted":
        r[40], r[41] = r[41], r[40]
    elif defect == "duplicate":
        r[41] = r[40]
    else:
        r[-1] = K
    cols[9] = r
    rp = np.zeros(17, np.int64)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols)
    v = rng.standard_normal(ci.size).astype(np.float32)
    with pytest.raises(hp.HrpbError) as e:
        gpu_build(16, K, rp, ci, v)
    assert e.value.status == 2


def test_builder_rejects_invalid_csr():
    M, K = 40, 50
    rp, ci, v = rand_csr(M, K, 0.2, 1)
    bad = []
    c2 = ci.copy(); c2[rp[3]], c2[rp[3] + 1] = c2[rp[3] + 1], c2[rp[3]]; bad.append((rp, c2))   # unsorted
    c3 = ci.copy(); c3[rp[5] + 1] = c3[rp[5]]; bad.append((rp, c3))                             # duplicate
    c4 = ci.copy(); c4[7] = K; bad.append((rp, c4))                                             # out of range
    r5 = rp.copy(); r5[10], r5[11] = r5[11], r5[10]; bad.append((r5, ci))                       # non-monotone
    for i, (r, c) in enumerate(bad):
        assert r[1 + 10] >= 0
        with pytest.raises(hp.HrpbError) as e:
            gpu_build(M, K, r, c, v)
        assert e.value.status == 2, i
    with pytest.raises(hp.HrpbError) as e:   # row_ptr[M] != nnz
        hp.build(dev(rp), dev(ci[:-1]), dev(v[:-1]), M, K)
    assert e.value.status == 2



@pytest.mark.parametrize("path", ["narrow", "wide", "wsort", "merge", "hub"])
@pytest.mark.parametrize("defect", ["unsorted", "duplicate"])
def test_builder_rejects_invalid_csr_every_ranking_path(path, defect):
    # one TM = 16 panel per case, shaped for each ranking path of the builder: warp byte map (span < 768), warp
    # bitmap (span < 8192), warp sort (wide, <= 256 entries), CTA merge ranking (wide, scattered, <= 2048
    # entries) and the hub path (> 2048 entries); one row then gets swapped or repeated columns
    rng = np.random.default_rng(7)
    per_row, span = {"narrow": (8, 600), "wide": (8, 6000), "wsort": (8, 10 ** 6), "merge": (60, 10 ** 6),
                     "hub": (200, 10 ** 6)}[path]
    K = 10 ** 6 + 7
    cols = [np.sort(rng.choice(span, per_row, replace=False)).astype(np.int32) for _ in range(16)]
    r = cols[5].copy()
    if defect == "unsorted":
        r[2], r[3] = r[3], r[2]
    else:
        r[3] = r[2]
    cols[5] = r
    rp = np.zeros(17, np.int64)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols)
    v = rng.standard_normal(ci.size).astype(np.float32)
    with pytest.raises(hp.HrpbError) as e:
        gpu_build(16, K, rp, ci, v)
    assert e.value.status == 2
    ok = [np.sort(rng.choice(span, per_row, replace=False)).astype(np.int32) for _ in range(16)]
    ci2 = np.concatenate(ok)  # the same shape, valid: bit-exact
    assert_same_hrpb(gpu_build(16, K, rp, ci2, v), oracle.csr_to_hrpb(16, K, rp, ci2, v), path)

# --------------------------------------------------------------------------- SpMM (S1..S5)
@pytest.mark.parametrize("N", [1, 8, 31, 32, 33, 100, 128, 200, 256, 384, 512, 520])
def test_spmm_exact_bitwise_widths(N):
    w = synth.make("c1", scale=2, N=N)  # 1024 x 1024, 1%, exact-mode integers
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    Cref = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B)
    check_exact(C, Cref, f"N={N}")


def test_spmm_exact_config1_full():
    w = synth.make("c1")  # BASELINE configs[0]: 4096^2, 1%, N = 32, exact mode
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(C, oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B), "c1")


@pytest.mark.parametrize("name,scale,N", [("c2a", 4, 128), ("c2b", 4, 128), ("c3", 7, 256), ("c3p", 7, 256),
                                          ("c4", 5, 512), ("c5", 3, 32), ("c5", 3, 64), ("c5", 3, 512)])
def test_spmm_float_tolerance(name, scale, N):
    w = synth.make(name, scale=scale, N=N)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B, with_bound=True)
    check_float(C, Cref, S, f"{name}/{N}")


@pytest.mark.parametrize("name,scale", [("c2a", 4), ("c3", 7), ("c5", 3)])
def test_spmm_exact_mode_other_structures(name, scale):
    w = synth.make(name, scale=scale, N=64, mode=synth.EXACT)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(C, oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B), name)


def test_spmm_edge_cases():
    rng = np.random.default_rng(3)
    # empty rows / empty panels are zeroed, C fully overwritten; M not a multiple of 16
    M, K, N = 53, 70, 48
    rp2 = np.zeros(M + 1, np.int64)
    # rows 20..35 emptied (panel 1 fully empty)
    r0, c0, v0 = rand_csr(M, K, 0.05, 7)
    cnt = np.diff(r0); cnt[20:36] = 0
    rp2[1:] = np.cumsum(cnt)
    ci2 = np.concatenate([c0[r0[i]:r0[i + 1]] if cnt[i] else c0[0:0] for i in range(M)]).astype(np.int32)
    v2 = np.concatenate([v0[r0[i]:r0[i + 1]] if cnt[i] else v0[0:0] for i in range(M)]).astype(np.float32)
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    A = gpu_build(M, K, rp2, ci2, v2)
    Cd = torch.full((M, N), float("nan"), device="cuda")
    hp.spmm(A, dev(B), out=Cd)
    check_exact(Cd.cpu().numpy(), oracle.csr_spmm(M, K, rp2, ci2, v2, B), "empty panel")
    # all-empty matrix
    A0 = gpu_build(M, K, np.zeros(M + 1, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    Cd = torch.full((M, N), float("nan"), device="cuda")
    hp.spmm(A0, dev(B), out=Cd)
    assert not Cd.cpu().numpy().any()
    # N = 0 is a no-op; dimension mismatch
    hp.spmm(A, dev(np.zeros((K, 0), np.float32)))
    with pytest.raises(hp.HrpbError) as e:
        hp.hrpb._check(hp.hrpb.lib().hrpb_spmm(A.handle, dev(B).data_ptr(), Cd.data_ptr(), M + 1, K, N, None),
                       "hrpb_spmm")
    assert e.value.status == 3


def test_spmm_hub_panel_and_dense_panel():
    rng = np.random.default_rng(11)
    M, K, N = 48, 20000, 96
    cols = [np.sort(rng.choice(K, rng.integers(1, 4000), replace=False)).astype(np.int32) for _ in range(M)]
    rp = np.zeros(M + 1, np.int64); rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols)
    v = rng.choice(np.array([-2, -1, 1, 2], np.float32), size=ci.shape[0])
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    A = gpu_build(M, K, rp, ci, v)
    assert_same_hrpb(A, oracle.csr_to_hrpb(M, K, rp, ci, v), "hub")
    check_exact(hp.spmm(A, dev(B)).cpu().numpy(), oracle.csr_spmm(M, K, rp, ci, v, B), "hub")


def test_spmm_unaligned_B_pointer():
    w = synth.make("c1", scale=3, N=20)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    big = torch.zeros(w.K * w.N + 1, device="cuda")
    Bd = big[1:].view(w.K, w.N)
    Bd.copy_(dev(B))
    C = torch.empty((w.M, w.N), device="cuda")
    hp.hrpb._check(hp.hrpb.lib().hrpb_spmm(A.handle, Bd.data_ptr(), C.data_ptr(), w.M, w.K, w.N, None), "spmm")
    torch.cuda.synchronize()
    check_exact(C.cpu().numpy(), oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B), "unaligned")


def test_host_entry_point_matches_device_path():
    w = synth.make("c5", scale=4, N=64)
    B = w.B()
    C = hp.build_spmm_host(w.row_ptr, w.col_idx, w.vals, B, w.M, w.K)
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B, with_bound=True)
    check_float(C, Cref, S, "host path")
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    Cd = hp.spmm(A, dev(B)).cpu().numpy()
    check_float(Cd, Cref, S, "device path")
    # the host path runs the SpMM in 16 panel-range launches, whose S1 work split (and hence the order in which a
    # split panel's partial tiles are added) differs from the single launch: equal within the bound, and each
    # path is deterministic
    C2 = hp.build_spmm_host(w.row_ptr, w.col_idx, w.vals, B, w.M, w.K)
    assert np.array_equal(C.view(np.uint32), C2.view(np.uint32))


def test_spmm_deterministic():
    w = synth.make("c3", scale=7, N=128)
    B = dev(w.B())
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    c1 = hp.spmm(A, B).cpu().numpy()
    c2 = hp.spmm(A, B).cpu().numpy()
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))


# --------------------------------------------------------------------------- TM > 16 panels (NEXT-1)
@pytest.mark.parametrize("tm,tk", [(32, 16), (64, 16), (128, 16), (16, 32), (32, 32), (64, 32)])
@pytest.mark.parametrize("N", [8, 128, 200, 512])
def test_spmm_exact_tm(tm, tk, N):
    w = synth.make("c1", scale=2, N=N)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm, tk=tk)
    assert A.tm == tm and A.tk == tk
    check_exact(hp.spmm(A, dev(B)).cpu().numpy(), oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B),
                f"tm={tm} tk={tk} N={N}")


@pytest.mark.parametrize("tm,tk", [(32, 16), (64, 16), (128, 16), (16, 32), (64, 32)])
@pytest.mark.parametrize("name,scale,N", [("c2a", 4, 128), ("c3", 7, 256), ("c5", 3, 64)])
def test_spmm_float_tm(tm, tk, name, scale, N):
    w = synth.make(name, scale=scale, N=N)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm, tk=tk)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B, with_bound=True)
    check_float(C, Cref, S, f"{name} tm={tm} tk={tk}")


# --------------------------------------------------------------------------- pipelined host entry point
@pytest.mark.parametrize("name,scale,N,tm,tk", [
    ("c2a", 6, 128, 64, 16),   # banded: C chunks start while later B chunks are still in flight
    ("c2a", 6, 100, 16, 16),   # N % 4 != 0: whole-matrix fallback after all of B
    ("c3", 8, 64, 32, 32),     # power law, TK = 32, hub columns anywhere in B
    ("c1", 3, 8, 16, 16),      # fewer panels than C chunks
])
def test_host_entry_pipelined_exact(name, scale, N, tm, tk):
    w = synth.make(name, scale=scale, N=N, mode=synth.EXACT)
    B = w.B()
    C = hp.build_spmm_host(w.row_ptr, w.col_idx, w.vals, B, w.M, w.K, tm=tm, tk=tk)
    check_exact(C, oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B), f"host {name} N={N} {tm}x{tk}")


def test_host_entry_empty_and_zero_rows():
    M, K, N = 300, 200, 16
    rp = np.zeros(M + 1, np.int64)
    C = hp.build_spmm_host(rp, np.zeros(0, np.int32), np.zeros(0, np.float32), np.ones((K, N), np.float32), M, K)
    assert C.shape == (M, N) and not C.any()


# --------------------------------------------------------------------------- S1: split big panels + fix-up
@pytest.mark.parametrize("tm", [16, 64, 128])
@pytest.mark.parametrize("N", [32, 300])
def test_spmm_split_hub_panels(tm, N):
    """A few hub panels each worth many CTAs' shares among thousands of small ones: the hubs are split between
    CTAs (partial tiles in the workspace, summed by k_spmm_fixup in CTA order). Exact mode, so C is bit-exact
    whatever the split; repeated calls are bitwise identical (deterministic fix-up order)."""
    rng = np.random.default_rng(5)
    M, K = 128 * 400, 30000
    lens = rng.integers(0, 6, M)
    for r in (tm * 7, tm * 7 + 3, tm * 200 + 1, M - 1):  # hub rows (two in one panel)
        lens[r] = 12000
    cols = [np.sort(rng.choice(K, n, replace=False)).astype(np.int32) for n in lens]
    rp = np.zeros(M + 1, np.int64); rp[1:] = np.cumsum(lens)
    ci = np.concatenate(cols)
    v = rng.choice(np.array([-2, -1, 1, 2], np.float32), size=ci.shape[0])
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    A = gpu_build(M, K, rp, ci, v, tm=tm)
    c1 = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(c1, oracle.csr_spmm(M, K, rp, ci, v, B), f"split hubs tm={tm} N={N}")
    c2 = hp.spmm(A, dev(B)).cpu().numpy()
    assert np.array_equal(c1.view(np.uint32), c2.view(np.uint32))


# --------------------------------------------------------------------------- fused device entry point
@pytest.mark.parametrize("tm", [16, 64])
def test_build_spmm_fused_matches_separate_calls(tm):
    w = synth.make("c2a", scale=6, N=128)
    B = dev(w.B())
    C1, A, (bms, sms) = hp.build_spmm(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), B, w.M, w.K, tm=tm, keep=True)
    assert bms > 0 and sms > 0
    assert_same_hrpb(A, oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm), "fused build")
    C2 = hp.spmm(gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm), B)
    assert torch.equal(C1.view(torch.int32), C2.view(torch.int32))   # same kernels, same launch configuration
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, w.B(), with_bound=True)
    check_float(C1.cpu().numpy(), Cref, S, "fused")


def test_build_spmm_fused_reports_invalid_csr():
    rp = np.array([0, 2, 3], np.int64)
    ci = np.array([5, 1, 0], np.int32)  # row 0 unsorted
    v = np.ones(3, np.float32)
    with pytest.raises(hp.HrpbError, match="INVALID_CSR"):
        hp.build_spmm(dev(rp), dev(ci), dev(v), torch.ones((8, 4), device="cuda"), 2, 8)


def test_build_spmm_graph_replay_exact():
    """Repeated identical hrpb_build_spmm calls on a side stream: call 1 eager, call 2 captured into a CUDA graph,
    calls 3+ replay it. Every result bit-exact (exact mode); a changed argument falls back to an eager call."""
    w = synth.make("c1", scale=1, N=64, mode=synth.EXACT)
    Cref = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, w.B())
    rp, ci, v, B = dev(w.row_ptr), dev(w.col_idx), dev(w.vals), dev(w.B())
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        C = torch.empty((w.M, w.N), device="cuda")
        for k in range(5):
            C.fill_(float("nan"))
            hp.build_spmm(rp, ci, v, B, w.M, w.K, out=C, stream=side)
            side.synchronize()
            check_exact(C.cpu().numpy(), Cref, f"call {k}")
        C2 = torch.empty_like(C)  # new output pointer: the plan is rebuilt
        hp.build_spmm(rp, ci, v, B, w.M, w.K, out=C2, stream=side)
        side.synchronize()
        check_exact(C2.cpu().numpy(), Cref, "changed out")


def test_build_spmm_async_replays_exact_and_deferred_errors():
    """hrpb_build_spmm_async: once graph-replayed, calls return without synchronizing. Results bit-exact (exact
    mode) after the stream syncs; an invalid CSR written into the same buffers is reported by the next
    hrpb_sync_status (and only once); valid input afterwards reports success again."""
    w = synth.make("c1", scale=1, N=64, mode=synth.EXACT)
    Cref = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, w.B())
    rp, ci, v, B = dev(w.row_ptr), dev(w.col_idx), dev(w.vals), dev(w.B())
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        C = torch.empty((w.M, w.N), device="cuda")
        for k in range(6):
            C.fill_(float("nan"))
            hp.build_spmm_async(rp, ci, v, B, w.M, w.K, C, stream=side)
            build_ms, spmm_ms = hp.sync_status(side)
            assert build_ms > 0 and spmm_ms > 0
            check_exact(C.cpu().numpy(), Cref, f"async call {k}")
        for _ in range(4):  # back to back, one sync at the end
            hp.build_spmm_async(rp, ci, v, B, w.M, w.K, C, stream=side)
        hp.sync_status(side)
        check_exact(C.cpu().numpy(), Cref, "back-to-back async calls")
        r = int(w.row_ptr[3])
        bad = w.col_idx.copy()
        bad[r], bad[r + 1] = bad[r + 1], bad[r]  # unsorted row, same buffers (the graph is replayed)
        ci.copy_(torch.from_numpy(bad).cuda())
        hp.build_spmm_async(rp, ci, v, B, w.M, w.K, C, stream=side)  # returns before the device has checked
        with pytest.raises(hp.HrpbError) as e:
            hp.sync_status(side)
        assert e.value.status == 2
        hp.sync_status(side)  # reported once
        ci.copy_(torch.from_numpy(w.col_idx).cuda())
        hp.build_spmm_async(rp, ci, v, B, w.M, w.K, C, stream=side)
        hp.sync_status(side)
        check_exact(C.cpu().numpy(), Cref, "after the error")
        with pytest.raises(hp.HrpbError) as e:  # the synchronous replay reports its own error directly
            ci.copy_(torch.from_numpy(bad).cuda())
            hp.build_spmm(rp, ci, v, B, w.M, w.K, out=C, stream=side)
        assert e.value.status == 2
        hp.sync_status(side)  # ... and not again here


@pytest.mark.parametrize("seed", range(6))
def test_spmm_split_boundaries_everywhere(seed):
    """S1 with epilogue-weighted units: panels of 1..250 blocks so that CTA boundaries fall in every kind of place
    (block units, a big panel's epilogue units, panel starts); exact mode, bit-exact against the oracle."""
    rng = np.random.default_rng(100 + seed)
    P, K, N = 96, 8192, 64
    rows, cols = [], []
    for p in range(P):
        nact = int(rng.choice([1, 5, 16, 40, 300, 1200, 4000])) if rng.random() < 0.7 else int(rng.integers(1, 4000))
        act = np.sort(rng.choice(K, nact, replace=False))
        for r in range(16):
            k = int(rng.integers(0, min(nact, 40) + 1))
            c = np.sort(rng.choice(act, k, replace=False)) if k else np.zeros(0, np.int64)
            if r == 0:
                c = act  # every active column appears in the panel
            cols.append(c.astype(np.int32))
    M = len(cols)
    rp = np.zeros(M + 1, np.int64)
    rp[1:] = np.cumsum([len(c) for c in cols])
    ci = np.concatenate(cols)
    v = rng.choice(np.array([-2, -1, 1, 2], np.float32), ci.size)
    Bh = rng.integers(-2, 3, (K, N)).astype(np.float32)
    A = gpu_build(M, K, rp, ci, v)
    C = hp.spmm(A, dev(Bh))
    check_exact(C.cpu().numpy(), oracle.csr_spmm(M, K, rp, ci, v, Bh), f"seed {seed}")


# --------------------------------------------------------------------------- tile choice, staging alternatives
def test_unsupported_tile_pair_rejected():
    """(TM, TK) = (128, 32) would need 64 brick slots per block (the decoder gives one lane per slot): rejected by
    every entry point before any work, like any other unsupported pair."""
    w = synth.make("c1", scale=3, N=8)
    for tm, tk in [(128, 32), (48, 16), (16, 8)]:
        with pytest.raises(hp.HrpbError) as e:
            gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm, tk=tk)
        assert e.value.status == 1
        with pytest.raises(hp.HrpbError) as e:
            hp.build_spmm(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), dev(w.B()), w.M, w.K, tm=tm, tk=tk)
        assert e.value.status == 1
        with pytest.raises(hp.HrpbError) as e:
            hp.build_spmm_host(w.row_ptr, w.col_idx, w.vals, w.B(), w.M, w.K, tm=tm, tk=tk)
        assert e.value.status == 1


@pytest.mark.parametrize("name,scale,want", [("c2a", 3, 64), ("c2b", 3, 64), ("c3", 6, 16), ("c4", 4, 16),
                                             ("c5", 2, 16), ("c1", 0, 16)])
def test_auto_tm_choice_and_parity(name, scale, want):
    """tm = 0: the library picks TM from a sampled B1 pass (DESIGN.md NEXT-1) -- the TM the measured sweep found
    fastest for each structure -- and the result is the oracle's HRPB at that TM, C within the tolerance."""
    w = synth.make(name, scale=scale)
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=0)
    assert A.tm == want, (name, A.tm)
    assert_same_hrpb(A, oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=A.tm), f"{name} auto")
    B = w.B()
    C = hp.spmm(A, dev(B)).cpu().numpy()
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B, with_bound=True)
    if w.mode == synth.EXACT:
        check_exact(C, Cref, f"{name} auto")
    else:
        check_float(C, Cref, S, f"{name} auto")


@pytest.fixture
def gather4(monkeypatch):
    monkeypatch.setenv("HRPB_GATHER", "0")  # S3 through TMA tile::gather4 instead of cp.async (read per call)
    yield


@pytest.mark.parametrize("tm", [16, 64, 128])
@pytest.mark.parametrize("N", [8, 33, 128, 256, 520])
def test_spmm_gather4_exact(gather4, tm, N):
    w = synth.make("c1", scale=2, N=N)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm)
    check_exact(hp.spmm(A, dev(B)).cpu().numpy(), oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B),
                f"gather4 tm={tm} N={N}")


@pytest.mark.parametrize("name,scale,N", [("c3", 7, 256), ("c5", 3, 64), ("c2a", 4, 100)])
def test_spmm_gather4_float(gather4, name, scale, N):
    w = synth.make(name, scale=scale, N=N)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B, with_bound=True)
    check_float(C, Cref, S, f"gather4 {name}")


def test_free_orders_after_spmm_on_other_streams():
    """hrpb_free right after an SpMM on another stream (no synchronization): the release waits for that stream
    (events recorded by hrpb_spmm), so the pool cannot hand the arrays to a new build while they are read."""
    w = synth.make("c5", scale=3, N=256, mode=synth.EXACT)
    B = dev(w.B())
    Cref = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, w.B())
    s2 = torch.cuda.Stream()
    for _ in range(3):
        A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
        C = torch.empty((w.M, w.N), device="cuda")
        hp.spmm(A, B, out=C, stream=s2)
        A.free()  # no sync
        junk = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, np.full_like(w.vals, 7.0))  # reuses pool memory
        s2.synchronize()
        check_exact(C.cpu().numpy(), Cref, "spmm vs free on another stream")
        junk.free()


@pytest.fixture
def dyn_s1(monkeypatch):
    monkeypatch.setenv("HRPB_DYN_S1", "1")  # dynamic S1 shares (read per call) on matrices below its size threshold


@pytest.mark.parametrize("tm", [16, 32])
@pytest.mark.parametrize("name,scale,N", [("c3", 9, 256), ("c3p", 9, 64), ("c5", 5, 128), ("c2a", 7, 520)])
def test_spmm_dynamic_s1_shares(dyn_s1, name, scale, N, tm):
    """Dynamic S1 (16 shares per SM claimed in order, split panels across shares through the fix-up): exact mode
    bit-identical to the oracle, float mode within tolerance."""
    w = synth.make(name, scale=scale, N=N, mode=synth.EXACT)
    B = w.B()
    A = gpu_build(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(C, oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B), f"{name} tm={tm}")
    wf = synth.make(name, scale=scale, N=N)
    Bf = wf.B()
    Af = gpu_build(wf.M, wf.K, wf.row_ptr, wf.col_idx, wf.vals, tm=tm)
    Cf = hp.spmm(Af, dev(Bf)).cpu().numpy()
    Cref, S = oracle.csr_spmm(wf.M, wf.K, wf.row_ptr, wf.col_idx, wf.vals, Bf, with_bound=True)
    check_float(Cf, Cref, S, f"{name} tm={tm} float")


def test_spmm_dynamic_s1_split_hubs(dyn_s1):
    """Hub panels much larger than a share: split over many shares (and CTAs), summed by the fix-up."""
    rng = np.random.default_rng(9)
    M, K, N = 16 * 3000, 40000, 128
    rp, ci, v = rand_csr(M, K, 0.0003, 5)
    dense = np.zeros((M, K), bool)
    for i in range(M):
        dense[i, ci[rp[i]:rp[i + 1]]] = True
    dense[[0, 1, 2, 17, 24000], :] = rng.random((5, K)) < 0.7
    rp = np.zeros(M + 1, np.int64); rp[1:] = np.cumsum(dense.sum(1))
    ci = np.nonzero(dense)[1].astype(np.int32)
    v = rng.choice(np.array([-2, -1, 1, 2], np.float32), size=ci.size).astype(np.float32)
    B = rng.choice(np.array([-1, 1, 2], np.float32), size=(K, N)).astype(np.float32)
    A = gpu_build(M, K, rp, ci, v)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(C, oracle.csr_spmm(M, K, rp, ci, v, B), "dynamic split hubs")


def test_spmm_dynamic_s1_hub_over_many_shares(dyn_s1):
    """One hub panel spread over more than 256 shares (the fix-up reduces its partial tiles in batches)."""
    rng = np.random.default_rng(21)
    M, K, N = 16 * 2400, 40000, 64
    rp, ci, v = rand_csr(M, K, 0.00005, 3)
    dense = np.zeros((M, K), bool)
    for i in range(M):
        dense[i, ci[rp[i]:rp[i + 1]]] = True
    dense[16 * 1200:16 * 1200 + 4, :] = rng.random((4, K)) < 0.9  # ~2300 blocks in one panel
    rp = np.zeros(M + 1, np.int64); rp[1:] = np.cumsum(dense.sum(1))
    ci = np.nonzero(dense)[1].astype(np.int32)
    v = rng.choice(np.array([-2, -1, 1, 2], np.float32), size=ci.size).astype(np.float32)
    B = rng.choice(np.array([-1, 1, 2], np.float32), size=(K, N)).astype(np.float32)
    A = gpu_build(M, K, rp, ci, v)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(C, oracle.csr_spmm(M, K, rp, ci, v, B), "hub over > 256 shares")
