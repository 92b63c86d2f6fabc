"""GPU parity of the NEXT-4 row reordering (hrpb_reorder_rows + hrpb_set_row_map): the permutation equals the
oracle's (O8) exactly, the permuted CSR is the input's rows in that order, and C = A.B computed from the reordered
HRPB with the row map equals the oracle's C of the ORIGINAL matrix (exact mode bit for bit, float mode within the
north-star tolerance) — through the static and the dynamic S1 paths, the split-panel fix-up and the sharded B."""
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


def reordered(w):
    perm, rp2, ci2, v2 = hp.reorder_rows(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), w.M, w.K)
    return perm, rp2, ci2, v2


@pytest.mark.parametrize("name,scale", [("c1", 0), ("c3", 6), ("c3p", 6), ("c4", 6), ("c5", 3), ("c2a", 6)])
def test_reorder_permutation_and_csr(name, scale):
    w = synth.make(name, scale=scale)
    perm, rp2, ci2, v2 = reordered(w)
    ref = oracle.reorder_rows(w.M, w.row_ptr, w.col_idx)
    assert np.array_equal(perm.cpu().numpy(), ref)
    rp = w.row_ptr
    deg = np.diff(rp)[ref]
    want_rp = np.zeros(w.M + 1, np.int64)
    want_rp[1:] = np.cumsum(deg)
    assert np.array_equal(rp2.cpu().numpy(), want_rp)
    idx = np.concatenate([np.arange(rp[r], rp[r + 1]) for r in ref]) if w.nnz else np.zeros(0, np.int64)
    assert np.array_equal(ci2.cpu().numpy(), w.col_idx[idx])
    assert np.array_equal(v2.cpu().numpy().view(np.uint32), w.vals[idx].view(np.uint32))


@pytest.fixture(params=["static", "dynamic"])
def s1_mode(request, monkeypatch):
    if request.param == "dynamic":
        monkeypatch.setenv("HRPB_DYN_S1", "1")
    return request.param


@pytest.mark.parametrize("tm", [16, 32, 64])
@pytest.mark.parametrize("name,scale,N", [("c3", 7, 256), ("c5", 3, 64), ("c4", 7, 36)])
def test_reordered_spmm_exact_original_order(s1_mode, name, scale, N, tm):
    w = synth.make(name, scale=scale, N=N, mode=synth.EXACT)
    B = w.B()
    perm, rp2, ci2, v2 = reordered(w)
    A = hp.build(rp2, ci2, v2, w.M, w.K, tm=tm)
    A.set_row_map(perm)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(C, oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B), f"{name} tm={tm} {s1_mode}")


def test_reordered_spmm_float_and_identity():
    w = synth.make("c3", scale=6, N=128)
    B = w.B()
    perm, rp2, ci2, v2 = reordered(w)
    A = hp.build(rp2, ci2, v2, w.M, w.K)
    A.set_row_map(perm)
    Bd = dev(B)
    C = hp.spmm(A, Bd).cpu().numpy()
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B, with_bound=True)
    check_float(C, Cref, S, "c3 reordered float")
    rps = -(-w.K // 3)
    with pytest.raises(hp.HrpbError):  # row maps are not instantiated for the row-sharded gather
        hp.spmm_sharded(A, [Bd[r:r + rps].clone() for r in range(0, w.K, rps)], rps)
    A.set_row_map(None)  # identity again: the permuted product
    Cp = hp.spmm(A, Bd).cpu().numpy()
    assert np.array_equal(Cp.view(np.uint32), C[perm.cpu().numpy()].view(np.uint32))


def test_reordered_split_hubs_and_empty_rows(monkeypatch):
    monkeypatch.setenv("HRPB_DYN_S1", "1")
    rng = np.random.default_rng(4)
    M, K, N = 16 * 400, 20000, 64
    rp, ci, v = rand_csr(M, K, 0.0004, 8)
    dense = np.zeros((M, K), bool)
    for i in range(M):
        dense[i, ci[rp[i]:rp[i + 1]]] = True
    dense[[5, 77, 3000], :] = rng.random((3, K)) < 0.8
    dense[100:400] = False  # empty rows
    rp = np.zeros(M + 1, np.int64); rp[1:] = np.cumsum(dense.sum(1))
    ci = np.nonzero(dense)[1].astype(np.int32)
    v = rng.choice(np.array([-2, -1, 1, 2], np.float32), size=ci.size).astype(np.float32)
    B = rng.choice(np.array([-1, 1, 2], np.float32), size=(K, N)).astype(np.float32)
    perm, rp2, ci2, v2 = hp.reorder_rows(dev(rp), dev(ci), dev(v), M, K)
    A = hp.build(rp2, ci2, v2, M, K)
    A.set_row_map(perm)
    C = hp.spmm(A, dev(B)).cpu().numpy()
    check_exact(C, oracle.csr_spmm(M, K, rp, ci, v, B), "reordered split hubs + empty rows")


def test_reorder_empty_matrix():
    rp = dev(np.zeros(65, np.int64))
    perm, rp2, ci2, v2 = hp.reorder_rows(rp, dev(np.zeros(0, np.int32)), dev(np.zeros(0, np.float32)), 64, 10)
    assert np.array_equal(rp2.cpu().numpy(), np.zeros(65, np.int64))
    A = hp.build(rp2, ci2, v2, 64, 10)
    A.set_row_map(perm)
    C = hp.spmm(A, dev(np.ones((10, 8), np.float32))).cpu().numpy()
    assert not C.any()
