"""Pins for the CPU oracle (oracle/): each check ties the oracle to something other than itself —
numpy's matmul, closed forms, SPEC/SURVEY worked examples (tests/golden), brute force over the
densified matrix, round trips, and injected corruptions the invariant checker must catch.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "hrpb_v1_examples.json")))


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


def to_csr(M, entries):
    entries = sorted(entries)
    rp = np.zeros(M + 1, np.int64)
    for r, _, _ in entries:
        rp[r + 1] += 1
    rp = np.cumsum(rp)
    ci = np.array([c for _, c, _ in entries], np.int32)
    v = np.array([x for _, _, x in entries], np.float32)
    return rp, ci, v


# ----------------------------------------------------------------------------- O1
def test_csr_validate_codes():
    rp, ci, v = to_csr(3, [(0, 1, 1.0), (0, 3, 1.0), (2, 0, 1.0)])
    assert oracle.csr_validate(3, 4, rp, ci) == 0
    assert oracle.csr_validate(3, 3, rp, ci) == 4               # column out of range
    bad = ci.copy(); bad[1] = 1
    assert oracle.csr_validate(3, 4, rp, bad) == 5              # duplicate in a row
    bad = ci.copy(); bad[0], bad[1] = 3, 1
    assert oracle.csr_validate(3, 4, rp, bad) == 5              # unsorted
    rpb = rp.copy(); rpb[1] = 3; rpb[2] = 1
    assert oracle.csr_validate(3, 4, rpb, ci) == 2              # non-monotone row_ptr


# ----------------------------------------------------------------------------- O2 / O3
@pytest.mark.parametrize("seed", range(6))
def test_csr_spmm_matches_numpy_exact(seed):
    rng = np.random.default_rng(100 + seed)
    M, K, N = rng.integers(1, 70, 3)
    rp, ci, v = rand_csr(M, K, rng.random() * 0.5, seed)
    B = rng.integers(-2, 3, (K, N)).astype(np.float32)
    C, S = oracle.csr_spmm(M, K, rp, ci, v, B, with_bound=True)
    A = oracle.densify(M, K, rp, ci, v)
    assert np.array_equal(C, A @ B.astype(np.float64))            # library matmul, exact on integers
    assert np.array_equal(S, np.abs(A) @ np.abs(B.astype(np.float64)))
    assert np.array_equal(oracle.dense_gemm(A, B), A @ B.astype(np.float64))  # O3 pinned to numpy too


def test_csr_spmm_special_cases():
    rng = np.random.default_rng(5)
    K, N = 37, 9
    B = rng.random((K, N)).astype(np.float32)
    rp = np.arange(K + 1, dtype=np.int64)
    ci = np.arange(K, dtype=np.int32)
    C = oracle.csr_spmm(K, K, rp, ci, np.ones(K, np.float32), B)
    assert np.array_equal(C, B.astype(np.float64))                # identity -> C = B
    perm = rng.permutation(K).astype(np.int32)
    C = oracle.csr_spmm(K, K, rp, perm, np.ones(K, np.float32), B)
    assert np.array_equal(C, B[perm].astype(np.float64))          # permutation -> permuted rows
    rp0 = np.zeros(K + 1, np.int64)
    C = oracle.csr_spmm(K, K, rp0, np.zeros(0, np.int32), np.zeros(0, np.float32), B)
    assert not C.any()                                            # empty -> 0


def test_csr_spmm_rows_subset_and_f32out():
    rng = np.random.default_rng(9)
    M, K, N = 50, 40, 7
    rp, ci, v = rand_csr(M, K, 0.2, 3, exact=False)
    B = rng.random((K, N)).astype(np.float32)
    full = oracle.csr_spmm(M, K, rp, ci, v, B)
    rows = np.array([49, 0, 17], np.int64)
    assert np.array_equal(oracle.csr_spmm(M, K, rp, ci, v, B, rows=rows), full[rows])
    c32, th = oracle.csr_spmm_f32out(M, rp, ci, v, B)
    assert th >= 1 and np.array_equal(c32, full.astype(np.float32))


# ----------------------------------------------------------------------------- O4 golden examples
def _gold_csr(case):
    M, K = case["M"], case["K"]
    if "rows" in case:
        return (M, K) + to_csr(M, [tuple(x) for x in case["rows"]])
    if "dense_value" in case:
        ents = [(r, c, float(1 + 16 * r + c)) for r in range(M) for c in range(K)]
        return (M, K) + to_csr(M, ents)
    ents = [(i, i, 1.0) for i in range(M)]
    return (M, K) + to_csr(M, ents)


@pytest.mark.parametrize("name", ["spec_16x20", "spec_dense16", "identity32"])
def test_convert_golden(name):
    case = GOLD[name]
    M, K, rp, ci, v = _gold_csr(case)
    h = oracle.csr_to_hrpb(M, K, rp, ci, v)
    assert h.blockedRowPtr.tolist() == case["blockedRowPtr"]
    assert h.activeCols.tolist() == case["activeCols"]
    assert h.sizePtr.tolist() == case["sizePtr"]
    assert h.packedBlocks.tobytes().hex() == case["packed_hex"]
    assert oracle.hrpb_check(h, ci.shape[0]) == (0, "")


def test_pattern_bit_order_matches_spec_examples():
    # encode({0,5,63}) = 0x8000000000000021: a single brick whose row-major positions
    # {0,5,63} = (r0,c0), (r1,c1), (r15,c3) hold entries; prefix_index examples.
    # (column 2 needs an entry too, else compaction moves column 3 left: entry (14,2) = bit 58)
    ents = [(0, 0, 1.0), (1, 1, 2.0), (14, 2, 4.0), (15, 3, 3.0)]
    rp, ci, v = to_csr(16, ents)
    h = oracle.csr_to_hrpb(16, 4, rp, ci, v)
    pat = int(np.frombuffer(h.packedBlocks[8:16].tobytes(), "<u8")[0])
    assert pat & ~(1 << 58) == int(GOLD["encode_example"]["pattern"], 16) and pat >> 58 & 1
    # the oracle stores values in ascending-bit order, so value index == prefix_index(pattern, bit)
    vals = np.frombuffer(h.packedBlocks[16:32].tobytes(), "<f4")
    assert vals.tolist() == [1.0, 2.0, 4.0, 3.0]
    for p_hex, pos, want in GOLD["prefix_example"]["cases"]:
        assert bin(int(p_hex, 16) & ((1 << pos) - 1)).count("1") == want


def test_convert_empty_and_ragged():
    h = oracle.csr_to_hrpb(40, 30, np.zeros(41, np.int64), np.zeros(0, np.int32), np.zeros(0, np.float32))
    assert h.blockedRowPtr.tolist() == [0, 0, 0, 0] and h.num_blocks == 0
    rp, ci, v = to_csr(37, [(36, 5, 2.0), (36, 29, -1.0), (0, 0, 1.0)])
    h = oracle.csr_to_hrpb(37, 30, rp, ci, v)
    assert h.blockedRowPtr.tolist() == [0, 1, 1, 2]                            # ceil(37/16) panels (R9)
    assert oracle.hrpb_check(h, 3)[0] == 0


# ----------------------------------------------------------------------------- O4 brute force
def brute_hrpb(M, K, rp, ci, v, tm=16, tk=16):
    """Independent tiny-input derivation from the dense matrix (numpy)."""
    A = oracle.densify(M, K, rp, ci, v)
    S = np.zeros((M, K), bool)
    for i in range(M):
        S[i, ci[rp[i]:rp[i + 1]]] = True
    P = (M + tm - 1) // tm
    brp, ac, blocks = [0], [], []
    for p in range(P):
        Sp = np.zeros((tm, K), bool); Ap = np.zeros((tm, K))
        rows = min(tm, M - p * tm)
        Sp[:rows] = S[p * tm:p * tm + rows]; Ap[:rows] = A[p * tm:p * tm + rows]
        act = np.nonzero(Sp.any(0))[0]
        nblk = -(-len(act) // tk)
        for j in range(nblk):
            cols = act[j * tk:(j + 1) * tk]
            ac += cols.tolist() + [K] * (tk - len(cols))
            Sb = np.zeros((tm, tk), bool); Ab = np.zeros((tm, tk))
            Sb[:, :len(cols)] = Sp[:, cols]; Ab[:, :len(cols)] = Ap[:, cols]
            bricks = []
            for bc in range(tk // 4):
                for br in range(tm // 16):
                    tile = Sb[16 * br:16 * br + 16, 4 * bc:4 * bc + 4].reshape(-1)
                    pat = sum(1 << int(i) for i in np.nonzero(tile)[0])
                    if pat:
                        vals = Ab[16 * br:16 * br + 16, 4 * bc:4 * bc + 4].reshape(-1)[tile]
                        bricks.append((bc, br, pat, vals))
            blocks.append(bricks)
        brp.append(brp[-1] + nblk)
    return brp, ac, blocks


def parse_blocks(h, tk=16):
    out = []
    nbc = tk // 4
    for b in range(h.num_blocks):
        blk = h.packedBlocks[int(h.sizePtr[b]):int(h.sizePtr[b + 1])].tobytes()
        colptr = list(blk[:nbc + 1]); nbr = colptr[-1]
        rows = list(blk[nbc + 1:nbc + 1 + nbr])
        hdr = -(-(nbc + 1 + nbr) // 8) * 8
        pats = np.frombuffer(blk[hdr:hdr + 8 * nbr], "<u8")
        nz = int(sum(bin(int(p)).count("1") for p in pats))
        vals = np.frombuffer(blk[hdr + 8 * nbr:hdr + 8 * nbr + 4 * nz], "<f4")
        bricks, off = [], 0
        for bc in range(nbc):
            for k in range(colptr[bc], colptr[bc + 1]):
                c = bin(int(pats[k])).count("1")
                bricks.append((bc, rows[k], int(pats[k]), vals[off:off + c].astype(np.float64)))
                off += c
        out.append(bricks)
    return out


@pytest.mark.parametrize("seed", range(12))
def test_convert_vs_bruteforce(seed):
    rng = np.random.default_rng(seed)
    M, K = int(rng.integers(1, 70)), int(rng.integers(1, 90))
    tm, tk = [(16, 16), (32, 16), (16, 32), (64, 16)][seed % 4]
    rp, ci, v = rand_csr(M, K, float(rng.choice([0.02, 0.1, 0.4, 0.9])), seed, exact=False)
    h = oracle.csr_to_hrpb(M, K, rp, ci, v, tm=tm, tk=tk)
    brp, ac, blocks = brute_hrpb(M, K, rp, ci, v, tm, tk)
    assert h.blockedRowPtr.tolist() == brp
    assert h.activeCols.tolist() == ac
    got = parse_blocks(h, tk)
    assert len(got) == len(blocks)
    for g, w in zip(got, blocks):
        assert [(a, b, c) for a, b, c, _ in g] == [(a, b, c) for a, b, c, _ in w]
        for (_, _, _, gv), (_, _, _, wv) in zip(g, w):
            assert np.array_equal(gv, wv)
    assert oracle.hrpb_check(h, ci.shape[0])[0] == 0


def test_convert_panel_range_equals_full_slice():
    w = synth.make("c5", scale=4)
    full = oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    p0, p1 = 7, 19
    part = oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals, p0=p0, p1=p1)
    b0, b1 = int(full.blockedRowPtr[p0]), int(full.blockedRowPtr[p1])
    assert np.array_equal(part.blockedRowPtr, full.blockedRowPtr[p0:p1 + 1] - b0)
    assert np.array_equal(part.activeCols, full.activeCols[b0 * 16:b1 * 16])
    s0, s1 = int(full.sizePtr[b0]), int(full.sizePtr[b1])
    assert np.array_equal(part.sizePtr, full.sizePtr[b0:b1 + 1] - s0)
    assert part.packedBlocks.tobytes() == full.packedBlocks[s0:s1].tobytes()


# ----------------------------------------------------------------------------- O5 / O6 / O7
@pytest.mark.parametrize("seed", range(20))
def test_round_trip(seed):
    rng = np.random.default_rng(1000 + seed)
    M, K = int(rng.integers(16, 300)), int(rng.integers(16, 300))
    dens = float(10 ** rng.uniform(-3, np.log10(0.3)))
    rp, ci, v = rand_csr(M, K, dens, seed, exact=False)
    h = oracle.csr_to_hrpb(M, K, rp, ci, v)
    rp2, ci2, v2 = oracle.hrpb_to_csr(h, ci.shape[0] + 1)
    assert np.array_equal(rp, rp2) and np.array_equal(ci, ci2) and np.array_equal(v, v2)
    code, msg = oracle.hrpb_check(h, ci.shape[0])
    assert code == 0, msg


def test_round_trip_keeps_explicit_zeros():
    rp, ci, v = to_csr(20, [(3, 4, 0.0), (3, 9, 1.5), (19, 0, 0.0)])
    h = oracle.csr_to_hrpb(20, 12, rp, ci, v)
    rp2, ci2, v2 = oracle.hrpb_to_csr(h, 10)
    assert ci2.tolist() == ci.tolist() and oracle.hrpb_check(h, 3)[0] == 0   # R11: structural


def _corrupt_cases(h):
    def mod(fn):
        import copy
        g = copy.deepcopy(h)
        fn(g)
        return g
    hdr = 8  # nbr <= 3 for the fixture below -> header 8 bytes
    yield "flip a pattern bit", mod(lambda g: g.packedBlocks.__setitem__(hdr, g.packedBlocks[hdr] ^ 0x40))
    yield "zero pattern", mod(lambda g: g.packedBlocks.__setitem__(slice(hdr, hdr + 8), 0))
    yield "swap activeCols", mod(lambda g: g.activeCols.__setitem__(slice(0, 2), g.activeCols[[1, 0]]))
    yield "blockedRowPtr", mod(lambda g: g.blockedRowPtr.__setitem__(1, g.blockedRowPtr[2] + 1))
    yield "pad byte", mod(lambda g: g.packedBlocks.__setitem__(7, 7))
    yield "colPtr", mod(lambda g: g.packedBlocks.__setitem__(1, 3))


def test_checker_catches_corruption():
    rp, ci, v = to_csr(40, [(0, 1, 1.0), (1, 2, 2.0), (3, 3, 3.0), (5, 9, 1.0), (17, 2, 4.0), (33, 7, 1.0)])
    h = oracle.csr_to_hrpb(40, 12, rp, ci, v)
    assert oracle.hrpb_check(h, 6)[0] == 0
    for what, g in _corrupt_cases(h):
        assert oracle.hrpb_check(g, 6)[0] != 0, what
    assert oracle.hrpb_check(h, 7)[0] != 0          # conservation: sum popcount = nnz


# One corruption per O6 return code, each asserting THAT code (oracle.c O6, codes 1-23). The fixture is
# hand-made so every corruption trips exactly the rule it targets (earlier rules stay satisfied).
def _o6_fixture():
    ents = [(0, 0, 1.0), (1, 1, 2.0), (2, 2, 3.0), (3, 3, 4.0)]          # panel 0, brick col 0: 4 bits
    ents += [(c % 16, c, float(c)) for c in range(4, 20)]                 # panel 0: 20 active cols, 2 blocks
    ents += [(16, 3, 1.0), (17, 5, 2.0), (20, 9, 3.0), (25, 21, 4.0), (31, 39, 5.0)]  # panel 1: 5 cols
    ents += [(32, 0, 1.0), (35, 7, 2.0), (39, 12, 3.0)]                   # panel 2 (ragged, rows 32..39)
    rp, ci, v = to_csr(40, ents)
    return oracle.csr_to_hrpb(40, 40, rp, ci, v), int(ci.shape[0])


def _blk(h, b):
    """byte offsets of block b's fields (HRPB-v1, TK = 16): colPtr, rows, patterns, values, end."""
    s = int(h.sizePtr[b])
    nbr = int(h.packedBlocks[s + 4])
    hdr = -(-(5 + nbr) // 8) * 8
    return {"colPtr": s, "rows": s + 5, "pat": s + hdr, "vals": s + hdr + 8 * nbr, "end": int(h.sizePtr[b + 1]),
            "nbr": nbr}


def _set_bit(h, off, bit, on=True):
    p = int(np.frombuffer(h.packedBlocks[off:off + 8].tobytes(), "<u8")[0])
    p = p | (1 << bit) if on else p & ~(1 << bit)
    h.packedBlocks[off:off + 8] = np.frombuffer(np.array([p], "<u8").tobytes(), np.uint8)


def _o6_cases():
    import copy
    h0, nnz = _o6_fixture()
    K = h0.K
    assert h0.blockedRowPtr.tolist() == [0, 2, 3, 4] and oracle.hrpb_check(h0, nnz) == (0, "")
    b0, b2, b3 = _blk(h0, 0), _blk(h0, 2), _blk(h0, 3)

    def mod(fn):
        g = copy.deepcopy(h0)
        fn(g)
        return g
    pk = lambda g: g.packedBlocks
    yield 1, mod(lambda g: setattr(g, "tm", 8)), nnz
    yield 2, mod(lambda g: g.blockedRowPtr.__setitem__(0, 1)), nnz
    yield 3, mod(lambda g: g.blockedRowPtr.__setitem__(1, 4)), nnz
    yield 4, mod(lambda g: g.sizePtr.__setitem__(0, 16)), nnz
    yield 5, mod(lambda g: g.sizePtr.__setitem__(1, 0)), nnz
    yield 6, mod(lambda g: g.sizePtr.__setitem__(1, g.sizePtr[1] + 8)), nnz
    yield 7, mod(lambda g: g.activeCols.__setitem__(2 * 16, K)), nnz           # sentinel, then a real column
    yield 8, mod(lambda g: g.activeCols.__setitem__(2 * 16, K + 5)), nnz       # column > K
    yield 9, mod(lambda g: g.activeCols.__setitem__(slice(0, 2), g.activeCols[[1, 0]])), nnz
    yield 10, mod(lambda g: g.activeCols.__setitem__(15, K)), nnz              # sentinel in a non-last block
    yield 11, mod(lambda g: pk(g).__setitem__(b0["colPtr"], 1)), nnz
    yield 12, mod(lambda g: pk(g).__setitem__(b0["colPtr"] + 1, 3)), nnz
    yield 13, mod(lambda g: pk(g).__setitem__(b0["rows"], 1)), nnz            # brick row >= TM/16
    yield 15, mod(lambda g: pk(g).__setitem__(slice(b0["pat"], b0["pat"] + 8), 0)), nnz
    yield 16, mod(lambda g: _set_bit(g, b2["pat"] + 8, 1)), nnz                # brick col 1, lc 1 is a sentinel
    yield 17, mod(lambda g: _set_bit(g, b3["pat"], 60)), nnz                   # row 32 + 15 >= M = 40
    yield 18, mod(lambda g: _set_bit(g, b0["pat"], 0, on=False)), nnz - 1      # full brick, popcount 3
    yield 19, mod(lambda g: g.sizePtr.__setitem__(4, g.sizePtr[4] + 16)), nnz
    yield 20, mod(lambda g: pk(g).__setitem__(b3["rows"] + 2, 7)), nnz          # header pad (nbr = 1)
    yield 21, mod(lambda g: pk(g).__setitem__(b3["end"] - 1, 7)), nnz           # tail pad
    yield 23, h0, nnz + 1                                                      # conservation
    # 14: rows not increasing inside a brick column (TM = 32: two brick rows)
    rp, ci, v = to_csr(40, [(0, 1, 1.0), (1, 2, 2.0), (3, 3, 3.0), (5, 9, 1.0), (17, 2, 4.0), (33, 7, 1.0)])
    h32 = oracle.csr_to_hrpb(40, 12, rp, ci, v, tm=32)
    assert oracle.hrpb_check(h32, 6) == (0, "")
    r = _blk(h32, 0)["rows"]
    assert h32.packedBlocks[r:r + 2].tolist() == [0, 1]
    g = copy.deepcopy(h32); g.packedBlocks[r + 1] = 0
    yield 14, g, 6
    # 22: a panel whose last block holds no real column (an empty block appended to a full one)
    rp, ci, v = to_csr(16, [(i, i, 1.0) for i in range(16)])
    h16 = oracle.csr_to_hrpb(16, 16, rp, ci, v)
    s = int(h16.sizePtr[1])
    g = oracle.Hrpb(16, 16, 16, 16, np.array([0, 2], np.uint32),
                    np.concatenate([h16.activeCols, np.full(16, 16, np.uint32)]),
                    np.array([0, s, s + 16], np.uint64), np.concatenate([h16.packedBlocks, np.zeros(16, np.uint8)]))
    yield 22, g, 16


def test_checker_every_code():
    got = {}
    for code, g, nnz in _o6_cases():
        c, msg = oracle.hrpb_check(g, nnz)
        assert c == code, (code, c, msg)
        got[code] = msg
    assert sorted(got) == list(range(1, 24))


def test_csr_validate_every_code():
    rp, ci, v = to_csr(3, [(0, 1, 1.0), (0, 3, 1.0), (2, 0, 1.0)])
    bad = rp.copy(); bad[0] = 1
    assert oracle.csr_validate(3, 4, bad, ci) == 1                               # row_ptr[0] != 0
    assert oracle.csr_validate(3, 4, rp, np.append(ci, 0).astype(np.int32)) == 3  # row_ptr[M] != nnz
    bad = ci.copy(); bad[2] = -1
    assert oracle.csr_validate(3, 4, rp, bad) == 4                               # negative column


def test_popcount_floor_tm16():
    # with TM = brick_m each real column of a brick has >= 1 nnz -> popcount >= 4
    w = synth.make("c2a", scale=8)
    h = oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals)
    ok = 0
    for bricks, b in zip(parse_blocks(h), range(h.num_blocks)):
        for bc, _, pat, _ in bricks:
            if all(h.activeCols[b * 16 + 4 * bc + j] != w.K for j in range(4)):
                assert bin(pat).count("1") >= 4
                ok += 1
    assert ok > 0


@pytest.mark.parametrize("tm", [16, 32])
def test_emulator_equals_csr_exact(tm):
    w = synth.make("c1", scale=3, N=24)
    B = w.B()
    h = oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm)
    assert np.array_equal(oracle.hrpb_spmm(h, B), oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, B))


# --------------------------------------------------------------------------- O8: NEXT-4 row reordering
def test_o8_reorder_hand_example():
    """DESIGN.md R25 key, worked by hand: degrees 2 / 0 / 5 / 1 -> log2 buckets 1 / 0 / 2 / 0, so row 2 (bucket 2)
    comes first, then row 0 (bucket 1); rows 1 and 3 share bucket 0 and row 3 (one column: a 24-bit hash) sorts
    before the empty row 1 (min-hash 2^24 - 1)."""
    rp = np.array([0, 2, 2, 7, 8], np.int64)
    ci = np.array([3, 9, 0, 1, 2, 3, 4, 5], np.int32)
    assert oracle.reorder_rows(4, rp, ci).tolist() == [2, 0, 3, 1]


@pytest.mark.parametrize("seed", range(4))
def test_o8_reorder_invariants(seed):
    """A permutation; degree buckets floor(log2(max(deg, 1))) never increase along it; rows with identical column
    sets in the same bucket keep their relative (row id) order."""
    rng = np.random.default_rng(seed)
    M, K = 300, 500
    rp, ci, _ = rand_csr(M, K, float(rng.choice([0.002, 0.02, 0.1])), seed)
    # duplicate some rows' column sets (identical keys)
    perm = oracle.reorder_rows(M, rp, ci)
    assert sorted(perm.tolist()) == list(range(M))
    deg = np.diff(rp)[perm]
    bucket = np.floor(np.log2(np.maximum(deg, 1))).astype(int)
    assert np.all(np.diff(bucket) <= 0)
    sets = {}
    for pos, r in enumerate(perm):
        sets.setdefault(tuple(ci[rp[r]:rp[r + 1]].tolist()), []).append(r)
    for rows in sets.values():
        assert rows == sorted(rows)


def test_o8_reorder_empty():
    assert oracle.reorder_rows(0, np.zeros(1, np.int64), np.zeros(0, np.int32)).size == 0
