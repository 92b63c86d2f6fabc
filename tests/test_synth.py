"""Synthetic input generators (synth/): canonical CSR, determinism, and the stated structure."""
import numpy as np
import pytest

import oracle
import synth


@pytest.mark.parametrize("name", synth.CONFIG_NAMES)
def test_configs_canonical_and_deterministic(name):
    scale = {"c1": 2, "c2a": 6, "c2b": 6, "c3": 9, "c3p": 9, "c4": 7, "c5": 3}[name]
    w = synth.make(name, scale=scale)
    assert oracle.csr_validate(w.M, w.K, w.row_ptr, w.col_idx) == 0
    w2 = synth.make(name, scale=scale)
    assert np.array_equal(w.row_ptr, w2.row_ptr) and np.array_equal(w.col_idx, w2.col_idx)
    assert np.array_equal(w.vals, w2.vals)
    if w.mode == synth.EXACT:
        assert set(np.unique(w.vals)) <= {-2.0, -1.0, 1.0, 2.0}
        assert set(np.unique(w.B())) <= {-2.0, -1.0, 0.0, 1.0, 2.0}
    else:
        assert w.vals.min() >= -1 and w.vals.max() < 1


def test_banded_structure():
    rp, ci = synth.banded(5000, 5000, 16, 32, seed=4)
    rows = np.repeat(np.arange(5000), np.diff(rp))
    assert np.all(np.abs(ci - rows) <= 32) and np.all(ci - rows >= -32) and np.all(ci - rows < 32)
    assert np.all(np.diff(rp)[40:-40] == 16)


def test_clustered_structure():
    rp, ci = synth.clustered(320, 4096, 4, 32, seed=2)
    for p in range(20):
        cols = ci[rp[16 * p]:rp[16 * p + 1]]
        assert len(cols) == 16 and np.all(cols.reshape(4, 4) % 4 == np.arange(4))
        for r in range(16 * p, 16 * p + 16):  # all rows of a panel share the clusters (dense 16x4)
            assert np.array_equal(ci[rp[r]:rp[r + 1]], cols)


def test_fem_blocks():
    rp, ci = synth.fem(10, 10, 8, seed=3)
    assert rp.shape[0] - 1 == 800
    for r in (0, 8 * 55 + 3, 799):
        cols = ci[rp[r]:rp[r + 1]]
        assert len(cols) % 8 == 0 and np.all(cols.reshape(-1, 8) % 8 == np.arange(8))


def test_rmat_power_law():
    rp, ci = synth.rmat(12, 16, seed=1)
    deg = np.diff(rp)
    assert deg.max() > 20 * max(1, np.median(deg))   # heavy tail
    assert oracle.csr_validate(4096, 4096, rp, ci) == 0


def test_dense_row_slices_match():
    full = synth.dense(50, 9, synth.FLOAT, seed=3)
    part = synth.dense(20, 9, synth.FLOAT, seed=3, r0=17)
    assert np.array_equal(full[17:37], part)
