"""GPU parity of hrpb_spmm_sharded (B row-sharded, each gathered row read from its shard).

The shards here are separate device allocations on one GPU (on a node they are peer-mapped allocations of the
other GPUs; the kernel addresses both the same way). Checks: float mode within the north-star tolerance of the
oracle, exact mode bit-identical to the oracle, and bit-identical to hrpb_spmm on the unsharded B (same
accumulation order), for shard counts 1..32, ragged last shards, every TM / TK and N widths with a ragged tail.
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


def shard(Bd, rps):
    """Row shards of B as separate allocations (clones): shard r = rows [r rps, min((r + 1) rps, K))."""
    K = Bd.shape[0]
    return [Bd[r:min(r + rps, K)].clone() for r in range(0, K, rps)]


@pytest.mark.parametrize("nsh", [1, 2, 3, 7, 8, 32])
@pytest.mark.parametrize("name,scale,N,tm", [("c3", 7, 256, 16), ("c2a", 4, 128, 64), ("c5", 3, 64, 16)])
def test_sharded_equals_unsharded_and_oracle(name, scale, N, tm, nsh):
    w = synth.make(name, scale=scale, N=N)
    B = w.B()
    A = hp.build(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), w.M, w.K, tm=tm)
    Bd = dev(B)
    rps = -(-w.K // nsh)
    shards = shard(Bd, rps)
    assert len(shards) == -(-w.K // rps)
    Cs = hp.spmm_sharded(A, shards, rps).cpu().numpy()
    Cu = hp.spmm(A, Bd).cpu().numpy()
    assert np.array_equal(Cs.view(np.uint32), Cu.view(np.uint32)), "sharded != unsharded"
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B, with_bound=True)
    check_float(Cs, Cref, S, f"{name}/{nsh}")


@pytest.mark.parametrize("tm,tk", [(16, 16), (32, 16), (64, 16), (128, 16), (16, 32), (64, 32)])
@pytest.mark.parametrize("N", [4, 36, 128, 260, 512])
def test_sharded_exact_ragged(tm, tk, N):
    rng = np.random.default_rng(tm * 1000 + tk * 10 + N)
    M, K = 700, 2900
    rp, ci, v = rand_csr(M, K, 0.02, tm + N)
    B = rng.choice(np.array([-2, -1, 1, 2], np.float32), size=(K, N)).astype(np.float32)
    A = hp.build(dev(rp), dev(ci), dev(v), M, K, tm=tm, tk=tk)
    Bd = dev(B)
    for rps in (K, 1000, 97, 91):  # 1, 3, 30, 32 shards; ragged last shard
        C = hp.spmm_sharded(A, shard(Bd, rps), rps).cpu().numpy()
        check_exact(C, oracle.csr_spmm(M, K, rp, ci, v, B), f"tm={tm} tk={tk} N={N} rps={rps}")


def test_sharded_split_hub_panels():
    """Panels larger than a CTA share (split between CTAs, k_spmm_fixup) with a sharded B."""
    rng = np.random.default_rng(5)
    M, K, N = 128 * 40, 30000, 64
    rp, ci, v = rand_csr(M, K, 0.0005, 11)
    # three dense hub rows spread over the matrix
    dense = np.zeros((M, K), bool)
    for i in range(M):
        dense[i, ci[rp[i]:rp[i + 1]]] = True
    dense[[3, 1700, 4000], :] = rng.random((3, K)) < 0.6
    rp = np.zeros(M + 1, np.int64); rp[1:] = np.cumsum(dense.sum(1))
    ci = np.nonzero(dense)[1].astype(np.int32)
    v = rng.choice(np.array([-1, 1, 2], np.float32), size=ci.size).astype(np.float32)
    B = rng.choice(np.array([-1, 1], np.float32), size=(K, N)).astype(np.float32)
    A = hp.build(dev(rp), dev(ci), dev(v), M, K)
    rps = 4096
    C = hp.spmm_sharded(A, shard(dev(B), rps), rps).cpu().numpy()
    check_exact(C, oracle.csr_spmm(M, K, rp, ci, v, B), "split hubs")


def test_sharded_rejects_bad_tables():
    import ctypes as C
    M, K, N = 64, 100, 8
    rp, ci, v = rand_csr(M, K, 0.1, 1)
    A = hp.build(dev(rp), dev(ci), dev(v), M, K)
    Bd = dev(np.ones((K, N), np.float32))
    out = torch.empty((M, N), device="cuda")
    lib = hp.hrpb.lib()

    def call(ptrs, nsh, rps, n=N):
        arr = (C.c_void_p * len(ptrs))(*ptrs)
        return lib.hrpb_spmm_sharded(A.handle, arr, nsh, rps, C.c_void_p(out.data_ptr()), M, K, n, None)

    p0, p1 = Bd.data_ptr(), Bd[50:].data_ptr()
    assert call([p0, p1], 2, 50) == 0
    assert call([p0, p1], 2, 40) == 1      # ceil(K / rps) != nshards
    assert call([p0 + 4, p1], 2, 50) == 1  # misaligned shard
    assert call([p0, 0], 2, 50) == 1       # null shard
    assert call([p0, p1], 2, 50, n=6) == 1  # N not a multiple of 4
    assert call([p0] * 33, 33, 4) == 1     # more than 32 shards
    assert lib.hrpb_spmm_sharded(A.handle, (C.c_void_p * 2)(p0, p1), 2, 50, C.c_void_p(out.data_ptr()), M, K + 1, N,
                                 None) == 3  # DIMENSION_MISMATCH
    with pytest.raises(ValueError):  # the binding checks shard shapes against rows_per_shard
        hp.spmm_sharded(A, [Bd[:60], Bd[60:]], 50)
