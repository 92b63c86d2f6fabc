"""Multi-GPU host logic on CPU: the row-panel partitioner and a world-size-2 gloo run of the sharded path
(broadcast of B + per-rank rows, computed with the CPU oracle in place of the CUDA kernels)."""
import os
import socket

import numpy as np
import pytest

import oracle
import synth
from paper_2504_06443_b200 import dist as hd


def test_shard_plan_contiguous_and_balanced():
    w = synth.make("c3", scale=8)  # power-law, skewed panels
    for world in (1, 2, 3, 4, 8):
        plan = hd.shard_plan(w.row_ptr, world)
        P = (w.M + 15) // 16
        assert plan[0].p0 == 0 and plan[-1].p1 == P
        for a, b in zip(plan, plan[1:]):
            assert a.p1 == b.p0
        wts = hd.panel_weights(w.row_ptr)
        per = [int(wts[s.p0:s.p1].sum()) for s in plan]
        assert sum(per) == w.nnz
        # each rank is within one (largest) panel of the ideal share
        assert max(per) - w.nnz / world <= wts.max() + 1


def test_shard_plan_more_ranks_than_panels():
    rp = np.array([0, 1, 2, 3], np.int64)  # 3 rows -> 1 panel
    plan = hd.shard_plan(rp, 4)
    assert sum(s.p1 - s.p0 for s in plan) == 1
    assert sum(s.nrows for s in plan) == 3


def test_slice_rows_rebases():
    w = synth.make("c5", scale=4)
    plan = hd.shard_plan(w.row_ptr, 3)
    rows = 0
    for s in plan:
        rp_l, ci_l, v_l = hd.slice_rows(w.row_ptr, w.col_idx, w.vals, s)
        assert rp_l[0] == 0 and rp_l[-1] == ci_l.shape[0] == v_l.shape[0]
        rows += s.nrows
    assert rows == w.M


def _free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = synth.make("c3", scale=9, N=24)
    B = torch.from_numpy(w.B()) if rank == 0 else torch.zeros((w.K, w.N), dtype=torch.float32)
    hd.broadcast_B(B)  # the path's only collective

    def cpu_compute(rp_l, ci_l, v_l, nrows, K, Bt):
        return oracle.csr_spmm(nrows, K, rp_l, ci_l, v_l, Bt.numpy())

    shard, C_local = hd.sharded_spmm(w.row_ptr, w.col_idx, w.vals, w.M, w.K, B, rank, world, compute=cpu_compute)
    np.save(os.path.join(out_dir, f"rank{rank}.npy"), C_local)
    np.save(os.path.join(out_dir, f"rank{rank}_rows.npy"), np.array([shard.row0, shard.nrows]))
    dist.barrier()
    dist.destroy_process_group()


def test_gloo_world2_sharded_equals_full(tmp_path):
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    w = synth.make("c3", scale=9, N=24)
    full = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, w.B())
    got = np.zeros_like(full)
    covered = 0
    for r in range(world):
        row0, nrows = np.load(tmp_path / f"rank{r}_rows.npy")
        got[row0:row0 + nrows] = np.load(tmp_path / f"rank{r}.npy")
        covered += nrows
    assert covered == w.M
    assert np.array_equal(got, full)  # same FP64 arithmetic per row -> identical


@pytest.mark.gpu
def test_sharded_cuda_path_single_process():
    """Both shards of a 2-way plan on one GPU through the C ABI, checked against the oracle."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    w = synth.make("c3", scale=8, N=64, mode=synth.EXACT)
    Bh = w.B()
    B = torch.from_numpy(Bh).cuda()
    full = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, Bh).astype(np.float32)
    for rank in range(2):
        shard, C = hd.sharded_spmm(w.row_ptr, w.col_idx, w.vals, w.M, w.K, B, rank, 2)
        assert np.array_equal(C.cpu().numpy(), full[shard.row0:shard.row0 + shard.nrows])


@pytest.mark.parametrize("world", [2, 4])
def test_bench_self_spawn_gloo(world):
    """`bench.py --gpus N` with WORLD_SIZE unset re-launches itself through torch.distributed.run (one process per
    rank, 127.0.0.1 rendezvous). --cpu-check runs that orchestration on CPU with gloo: shard_plan partition, the B
    broadcast, max/sum over ranks and rank 0's single JSON line; each rank's rows are checked against the oracle."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--cpu-check", "--gpus", str(world)],
                       capture_output=True, text=True, timeout=600, env=env, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 alone prints
    d = lines[0]
    assert d["world"] == world and d["parity"] is True and d["scaling"] == "strong"
    assert d["rows"] == d["M"] and d["nnz"] == d["total_nnz"]  # the shards cover the matrix exactly once


def test_shard_plan_explicit_weights():
    w = synth.make("c3", scale=8)
    P = (w.M + 15) // 16
    wts = np.random.default_rng(0).integers(0, 50, P)
    plan = hd.shard_plan(w.row_ptr, 4, 16, wts)
    per = [int(wts[s.p0:s.p1].sum()) for s in plan]
    assert plan[0].p0 == 0 and plan[-1].p1 == P and sum(per) == wts.sum()
    assert max(per) - wts.sum() / 4 <= wts.max() + 1
    with pytest.raises(ValueError):
        hd.shard_plan(w.row_ptr, 4, 16, wts[:-1])


def test_b_row_shards_cover_rows():
    for K in (0, 1, 7, 100, 4194304):
        for world in (1, 2, 3, 8):
            rps, rows = hd.b_row_shards(K, world)
            assert rows[0][0] == 0 and rows[-1][1] == K
            for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
                assert a1 == b0 and a0 <= a1
            nsh = -(-K // rps) if K else 1
            assert nsh <= world
            # the shards the kernel addresses: rank r < nsh holds rows [r rps, min((r + 1) rps, K))
            for r in range(nsh):
                assert rows[r] == (r * rps, min((r + 1) * rps, K))
            assert all(a == b for a, b in rows[nsh:]) or K == 0
