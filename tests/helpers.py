"""Shared test helpers: tolerance of the north star and oracle/GPU comparison utilities."""
import numpy as np

TOL_REL = 4.0 * 2.0 ** -11   # north star: |C - C_ref| <= 4 * 2^-11 * sum|a||b| + 1e-6
TOL_ABS = 1e-6


def check_float(C, Cref, S, what=""):
    C = np.asarray(C, np.float64)
    err = np.abs(C - Cref)
    bound = TOL_REL * S + TOL_ABS
    bad = err > bound
    if bad.any():
        i = np.argwhere(bad)[0]
        raise AssertionError(f"{what}: {int(bad.sum())} elements out of tolerance, first {tuple(i)}: "
                             f"got {C[tuple(i)]!r} want {Cref[tuple(i)]!r} bound {bound[tuple(i)]!r}")
    return float((err / np.maximum(bound, 1e-300)).max()) if err.size else 0.0


def check_exact(C, Cref, what=""):
    want = Cref.astype(np.float32)
    got = np.asarray(C, np.float32)
    if not np.array_equal(got.view(np.uint32), want.view(np.uint32)):
        bad = np.argwhere(got != want)
        raise AssertionError(f"{what}: {len(bad)} mismatches, first {tuple(bad[0]) if len(bad) else None}")


def rand_csr(M, K, density, seed, exact=True):
    rng = np.random.default_rng(seed)
    mask = rng.random((M, K)) < density
    rp = np.zeros(M + 1, np.int64)
    rp[1:] = np.cumsum(mask.sum(1))
    ci = np.nonzero(mask)[1].astype(np.int32)
    if exact:
        v = rng.choice(np.array([-2, -1, 1, 2], np.float32), size=ci.shape[0])
    else:
        v = (rng.random(ci.shape[0]) * 2 - 1).astype(np.float32)
    return rp, ci, v.astype(np.float32)
