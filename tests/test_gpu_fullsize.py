"""Full-size parity (BASELINE.json configs at their real sizes), in the configuration bench.py times.

The oracle cannot produce full outputs in seconds, so each case checks:
  * HRPB: the complete GPU arrays against the oracle invariant checker (O6), plus byte-exact equality of
    sampled panels against the oracle converter run on just those panels;
  * SpMM: sampled rows of C against the FP64 oracle (bit-exact in exact mode, the north-star tolerance
    in float mode), plus whole-matrix properties (finite, zero rows for empty rows).
"""
import numpy as np
import pytest

import oracle
import synth
from helpers import check_exact, check_float

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a B200", allow_module_level=True)

import paper_2504_06443_b200 as hp  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def sample_panels(P, k, seed):
    rng = np.random.default_rng(seed)
    base = [0, 1, P // 2, P - 1]
    return sorted(set(base + list(rng.choice(P, size=min(k, P), replace=False))))


def check_sampled_panels(A, w, tm, panels):
    brp, ac, sp, packed = A.to_host()
    for p in panels:
        ref = oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm, p0=p, p1=p + 1)
        b0, b1 = int(brp[p]), int(brp[p + 1])
        assert b1 - b0 == ref.num_blocks, f"panel {p}: block count"
        assert np.array_equal(ac[b0 * 16:b1 * 16], ref.activeCols), f"panel {p}: activeCols"
        s0, s1 = int(sp[b0]), int(sp[b1])
        assert np.array_equal(sp[b0:b1 + 1] - s0, ref.sizePtr), f"panel {p}: sizePtr"
        assert packed[s0:s1].tobytes() == ref.packedBlocks.tobytes(), f"panel {p}: packedBlocks"
    return brp, ac, sp, packed


def run_case(name, N, tm, mode=None, rows_sample=384, panels_sample=48, full_check=True):
    w = synth.make(name, N=N, mode=mode)
    A = hp.build(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), w.M, w.K, tm=tm)
    brp, ac, sp, packed = check_sampled_panels(A, w, tm, sample_panels(A.num_panels, panels_sample, 1))
    if full_check:
        h = oracle.Hrpb(w.M, w.K, tm, 16, brp, ac, sp, packed)
        code, msg = oracle.hrpb_check(h, w.nnz)
        assert code == 0, msg
    Bh = w.B()
    Bd = dev(Bh)
    C = hp.spmm(A, Bd)
    rng = np.random.default_rng(2)
    rows = np.unique(np.concatenate([[0, w.M - 1], rng.choice(w.M, rows_sample, replace=False)])).astype(np.int64)
    Cs = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, Bh, rows=rows, with_bound=True)
    if w.mode == synth.EXACT:
        check_exact(Cs, Cref, f"{name} tm={tm}")
    else:
        check_float(Cs, Cref, S, f"{name} tm={tm}")
    assert bool(torch.isfinite(C).all())
    empty = np.nonzero(np.diff(w.row_ptr) == 0)[0]
    if empty.size:
        e = torch.from_numpy(empty[:4096].astype(np.int64)).cuda()
        assert not bool(C[e].any())
    del C, Bd
    torch.cuda.empty_cache()


def test_config1_full_exact_all_rows():
    # configs[0]: 4096^2, 1%, N = 32, exact mode -> the whole C is compared bit for bit
    w = synth.make("c1")
    Bh = w.B()
    for tm in (16, 64):
        A = hp.build(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), w.M, w.K, tm=tm)
        C = hp.spmm(A, dev(Bh)).cpu().numpy()
        check_exact(C, oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, Bh), f"c1 tm={tm}")


@pytest.mark.parametrize("tm", [16, 64])
def test_config2a_banded_full(tm):  # configs[1] (bench workload; bench.py picks TM by its plan step)
    run_case("c2a", 128, tm)


@pytest.mark.parametrize("tm", [16, 64])
def test_config2b_clustered_full(tm):
    run_case("c2b", 128, tm)


def test_config3_rmat_full():  # configs[2]: R-MAT scale 22, N = 256 (hub panels exercise the bitmap path)
    run_case("c3", 256, 16, rows_sample=256, panels_sample=24)


def test_config3_rmat_exact_mode():  # exact mode on the power-law structure (row sums stay < 2^24)
    run_case("c3", 64, 16, mode=synth.EXACT, rows_sample=256, panels_sample=8, full_check=False)


def test_config3_rmat_static_s1(monkeypatch):  # the headline size through the static S1 kernel too
    monkeypatch.setenv("HRPB_STATIC_S1", "1")
    run_case("c3", 64, 16, mode=synth.EXACT, rows_sample=256, panels_sample=8, full_check=False)


def test_config4_uniform_dynamic_s1(monkeypatch):  # dynamic S1 forced below its size threshold, full size
    monkeypatch.setenv("HRPB_DYN_S1", "1")
    run_case("c4", 512, 16, rows_sample=256, panels_sample=8, full_check=False)


def test_config4_uniform_full():  # configs[3]: 2M^2, 8 nnz/row, N = 512
    run_case("c4", 512, 16, rows_sample=256, panels_sample=24)


@pytest.mark.parametrize("N", [32, 512])
def test_config5_fem_full(N):  # configs[4]: FEM 500K^2, N sweep
    run_case("c5", N, 16, rows_sample=256, panels_sample=24, full_check=(N == 32))


# --------------------------------------------------------------------------- whole-array HRPB at full size
@pytest.mark.parametrize("name,tm", [("c2a", 64), ("c2a", 16), ("c2b", 64), ("c4", 16), ("c5", 16)])
def test_full_size_hrpb_whole_array(name, tm):
    """Every byte of blockedRowPtr / activeCols / sizePtr / packedBlocks against the oracle converter run on the
    whole matrix (not sampled panels)."""
    w = synth.make(name)
    A = hp.build(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), w.M, w.K, tm=tm)
    ref = oracle.csr_to_hrpb(w.M, w.K, w.row_ptr, w.col_idx, w.vals, tm=tm)
    brp, ac, sp, packed = A.to_host()
    assert np.array_equal(brp, ref.blockedRowPtr)
    assert np.array_equal(ac, ref.activeCols)
    assert np.array_equal(sp, ref.sizePtr)
    assert packed.tobytes() == ref.packedBlocks.tobytes()


# --------------------------------------------------------------------------- the bench's exact step
def bench_step_check(name, want_tm, rows_sample=2048, hub_rows=64):
    """bench.py's step: hrpb_build_spmm_async with tm = 0 (library choice), graph-replayed back to back on a side
    stream, full-size inputs resident in HBM; C (after the replays) against the FP64 oracle on sampled rows plus
    the heaviest rows, within the north-star tolerance; every replay's CSR status clean."""
    w = synth.make(name)
    Bh = w.B()
    rp, ci, v, B = dev(w.row_ptr), dev(w.col_idx), dev(w.vals), dev(Bh)
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        C = torch.full((w.M, w.N), float("nan"), device="cuda")
        _, A, _ = hp.build_spmm(rp, ci, v, B, w.M, w.K, out=C, tm=0, stream=side, keep=True)
        assert A.tm == want_tm, A.tm
        A.free()
        for _ in range(3):  # eager, capture, replays
            hp.build_spmm(rp, ci, v, B, w.M, w.K, out=C, tm=0, stream=side)
        C.fill_(float("nan"))
        for _ in range(5):  # the timed loop: replays without host synchronization
            hp.build_spmm_async(rp, ci, v, B, w.M, w.K, C, tm=0, stream=side)
        hp.sync_status(side)
    rng = np.random.default_rng(5)
    heavy = np.argsort(np.diff(w.row_ptr))[-hub_rows:]
    rows = np.unique(np.concatenate([[0, w.M - 1], heavy, rng.choice(w.M, rows_sample, replace=False)])).astype(np.int64)
    Cs = C[torch.from_numpy(rows).cuda()].cpu().numpy()
    Cref, S = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, Bh, rows=rows, with_bound=True)
    check_float(Cs, Cref, S, f"bench step {name}")
    assert bool(torch.isfinite(C).all())


def test_bench_step_c3_full():
    bench_step_check("c3", 16)


def test_bench_step_c2a_full():
    bench_step_check("c2a", 64)
