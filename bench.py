#!/usr/bin/env python
"""bench.py — HRPB SpMM on B200 (the hot path of cuTeSpMM, arxiv 2504.06443).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one pass of the whole hot path over one batch of synthetic input: hrpb_build (CSR ->
HRPB on the GPU) + hrpb_spmm (S1-S5), inputs resident in HBM.
Workload (BASELINE.json configs[1], banded variant "c2a"): per rank a banded 2^20 x 2^20 slab,
16 distinct columns per row in [i-32, i+32), N = 128, float mode. With N GPUs the matrix is the
vertical stack of N such slabs sharing one B (weak scaling; row panels partitioned, B broadcast once
over NCCL at setup, no reduction — SURVEY §8(e)).

Metric: effective GFLOP/s = 2 * nnz * N / t (BASELINE.json metric), whole job.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

M0 = 1 << 20          # rows per rank slab (= K)
K0 = 1 << 20
NCOL = 128            # N
DEG, HALF_W = 16, 32
METRIC = "SpMM effective GFLOP/s (2*nnz*N/t) and % HBM/TF32 roofline"
UNIT = "GFLOP/s"
WORKLOAD = ("c2a: banded A, per-rank slab M=K=2^20, 16 distinct nnz/row uniform in [i-32,i+32), N=128, "
            "float mode (BASELINE configs[1], banded variant)")


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def make_slab(rank: int):
    rp, ci = synth.banded(M0, K0, DEG, HALF_W, seed=1, r0=rank * M0, shift=rank * M0)
    vals = synth.values_a(int(ci.shape[0]), synth.FLOAT, seed=2, e0=rank * M0 * DEG)
    return rp, ci, vals


def read_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, gpu_index: int):
        self.proc = None
        self.path = f"/tmp/hrpb_clocks_{os.getpid()}.csv"
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "samples": len(sm),
                "reasons": sorted(reasons)}


def ncu_traffic(kernel: str, workload_tag: str):
    """dram bytes (read + write) per launch of `kernel` from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(path))
        e = d.get(kernel, {})
        if str(e.get("workload", "")).split("_")[0] == workload_tag:  # (summaries may tag "c2a_tm64")
            return e.get("dram_bytes_per_launch")
    except Exception:
        pass
    return None


def measure_tf32_peak(torch):
    """cuBLAS fp32 GEMM with TF32 tensor cores, 8192^3, best of 5 (the TF32 roof MEASURED_PEAKS lacks)."""
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device="cuda")
    b = torch.randn(8192, 8192, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); a @ b; e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    del a, b
    torch.backends.cuda.matmul.allow_tf32 = False
    return 2 * 8192 ** 3 / best / 1e12


def cpu_baseline_oracle(rp, ci, vals, B, target_s=12.0, cap_s=30.0):
    """Oracle CSR SpMM (FP64 accumulate, fp32 out, OpenMP over rows) on the host cores; bounded sample:
    passes over the whole slab repeat until ~target_s seconds of CPU work have run (cap cap_s)."""
    import oracle
    M = rp.shape[0] - 1
    rows = M
    out = np.empty((rows, B.shape[1]), np.float32)
    oracle.csr_spmm_f32out(M, rp, ci, vals, B, 0, rows, out=out)  # first touch / thread start-up
    reps, th = 0, 1
    t = time.perf_counter()
    while True:
        _, th = oracle.csr_spmm_f32out(M, rp, ci, vals, B, 0, rows, out=out)
        reps += 1
        dt = time.perf_counter() - t
        if dt >= target_s or dt * (reps + 1) / reps > cap_s:
            break
    nnz_s = int(rp[rows] - rp[0])
    gf = 2.0 * nnz_s * B.shape[1] * reps / dt / 1e9
    return {"value": round(gf, 3), "unit": UNIT, "cores": int(th), "kind": "oracle",
            "sample": f"rows [0,{rows}) of the rank-0 c2a slab ({nnz_s} nnz), N={B.shape[1]}, x{reps}, "
                      f"{dt:.1f} s, FP64-accumulating CSR SpMM with fp32 output (oracle/oracle.c)"}


# ------------------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The tier's reference arm: the CPU oracle as it stands, on this box's host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    rp, ci, vals = make_slab(0)
    B = synth.dense(K0, NCOL, synth.FLOAT, seed=3)
    M = rp.shape[0] - 1
    total_steps = args.steps + args.warmup
    budget = 150.0  # seconds for the whole run
    # one reference step = oracle CSR->HRPB conversion + oracle CSR SpMM on a row sample (mirrors build+spmm)
    probe_rows = 16 * 256
    t = time.perf_counter()
    oracle.csr_to_hrpb(M, K0, rp, ci, vals, p0=0, p1=probe_rows // 16)
    oracle.csr_spmm_f32out(M, rp, ci, vals, B, 0, probe_rows)
    per_row = (time.perf_counter() - t) / probe_rows
    rows = int(max(16, min(M, budget / total_steps / max(per_row, 1e-12))) // 16 * 16)
    out = np.empty((rows, NCOL), np.float32)
    th = oracle.num_threads()

    def step():
        oracle.csr_to_hrpb(M, K0, rp, ci, vals, p0=0, p1=rows // 16)
        oracle.csr_spmm_f32out(M, rp, ci, vals, B, 0, rows, out=out)

    for _ in range(args.warmup):
        step()
    t = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t) / max(args.steps, 1)
    nnz_s = int(rp[rows])
    v = 2.0 * nnz_s * NCOL / dt / 1e9
    sample = (f"rows [0,{rows}) of the c2a slab ({nnz_s} nnz) per step: oracle CSR->HRPB (serial) + "
              f"oracle CSR SpMM (FP64 acc, OpenMP)")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "sample_rows": rows},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": th, "kind": "oracle", "sample": sample},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------ our arm
def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2504_06443_b200 as hp
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)

    rp, ci, vals = make_slab(rank)
    nnz = int(ci.shape[0])
    rp_d = torch.from_numpy(rp).to(dev)
    ci_d = torch.from_numpy(ci).to(dev)
    v_d = torch.from_numpy(vals).to(dev)
    # B: generated on rank 0, broadcast once over NCCL (north star: "B is broadcast once")
    if rank == 0:
        B_h = synth.dense(K0, NCOL, synth.FLOAT, seed=3)
        B_d = torch.from_numpy(B_h).to(dev)
    else:
        B_h = None
        B_d = torch.empty((K0, NCOL), dtype=torch.float32, device=dev)
    bcast_ms = None
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        dist.broadcast(B_d, src=0)
        e.record()
        torch.cuda.synchronize()
        bcast_ms = s.elapsed_time(e)
    C_d = torch.empty((M0, NCOL), dtype=torch.float32, device=dev)

    # a dedicated (non-default) stream: the library captures the repeated build + SpMM call into a CUDA graph,
    # which the legacy default stream does not allow
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    tm_plan = None
    if args.tm == 0:  # plan: time one build + spmm per candidate TM (untimed, like a library autotuner)
        tm_plan = {}
        for cand in (16, 32, 64):
            for it in range(3):
                s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s0.record(stream)
                hp.build_spmm(rp_d, ci_d, v_d, B_d, M0, K0, out=C_d, tm=cand, stream=stream)
                s1.record(stream)
                torch.cuda.synchronize()
            tm_plan[cand] = round(s0.elapsed_time(s1), 4)
        best = min(tm_plan, key=tm_plan.get)
        if world > 1:  # every rank uses rank 0's choice
            t = torch.tensor([best], device=dev)
            dist.broadcast(t, src=0)
            best = int(t.item())
        args.tm = best

    phase = []  # (build_ms, spmm_ms) per timed step, CUDA events recorded by the library on `stream`

    def step(timed=False):
        # hrpb_build_spmm: build + SpMM enqueued back to back, one synchronisation per step (phase times)
        _, _, ms = hp.build_spmm(rp_d, ci_d, v_d, B_d, M0, K0, out=C_d, tm=args.tm, stream=stream)
        if timed:
            phase.append(ms)

    def step_async():
        # hrpb_build_spmm_async: the same graph-replayed build + SpMM without the per-step host round trip; the
        # CSR status of every step is checked by hrpb_sync_status after the timed loop
        hp.build_spmm_async(rp_d, ci_d, v_d, B_d, M0, K0, C_d, tm=args.tm, stream=stream)

    for _ in range(max(args.warmup, 3)):
        step()
    for _ in range(8):  # phase times: synchronous steps (library CUDA events), outside the timed region
        step(timed=True)
    step_async()
    hp.sync_status(stream)
    torch.cuda.synchronize()
    # structural statistics for the roofline (from a built handle, outside the timed region)
    A = hp.build(rp_d, ci_d, v_d, M0, K0, tm=args.tm)
    torch.cuda.synchronize()
    brp, ac, sp, packed_h = A.to_host()
    NB, P, packed = A.num_blocks, A.num_panels, A.packed_bytes
    sum_nact = int(np.count_nonzero(ac != K0))
    bricks = int(packed_h[sp[:-1].astype(np.int64) + 4].astype(np.int64).sum())  # colPtr[4] = nbr per block (TK=16)
    alpha = nnz / max(1, 64 * bricks)  # brick density
    A.free()
    uniq = int(np.count_nonzero(np.bincount(ci, minlength=K0)))

    # ---------------------------------------------------------------- timed region
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = hp.launch_count()
    t0.record(stream)
    for k in range(args.steps):
        step_async()
    t1.record(stream)
    # raises if any timed step saw an invalid CSR; returns the phase times of the last timed step (the library's
    # CUDA events inside the replayed graph, on `stream`)
    last_phase = hp.sync_status(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = hp.launch_count() - launches0
    clk = clocks.stop()
    ms = t0.elapsed_time(t1) / max(args.steps, 1)
    # phase times: the last timed step's (inside the timed region) averaged with the 8 synchronous steps run
    # just before it (same graph, same launch configuration)
    build_ms = float(np.mean([p[0] for p in phase] + [last_phase[0]]))
    spmm_ms = float(np.mean([p[1] for p in phase] + [last_phase[1]]))
    stats = torch.tensor([ms, build_ms, spmm_ms, float(nnz)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, build_ms, spmm_ms, total_nnz = float(mx[0]), float(mx[1]), float(mx[2]), float(sm[3])
    else:
        total_nnz = float(nnz)
    flops = 2.0 * total_nnz * NCOL
    value = flops / (ms / 1e3) / 1e9

    # ---------------------------------------------------------------- e2e through the host C-ABI entry
    if B_h is None:
        B_h = B_d.cpu().numpy()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    rp_h, ci_h, v_h, Bp_h = pin(rp), pin(ci), pin(vals), pin(B_h)
    Cp_h = torch.empty((M0, NCOL), dtype=torch.float32).pin_memory()
    hp.build_spmm_host(rp_h, ci_h, v_h, Bp_h, M0, K0, out=Cp_h, tm=args.tm)  # warm
    e2e_steps = max(1, min(args.steps, 5))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(e2e_steps):
        hp.build_spmm_host(rp_h, ci_h, v_h, Bp_h, M0, K0, out=Cp_h, tm=args.tm)
    e.record(stream)
    torch.cuda.synchronize()
    e2e_ms = s.elapsed_time(e) / e2e_steps
    if world > 1:
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t[0])
    h2d = (M0 + 1) * 8 + nnz * 8 + K0 * NCOL * 4
    d2h = M0 * NCOL * 4

    if rank != 0:
        if dist is not None:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peaks = read_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy)"
    if not hbm:
        hbm, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    meta_bytes = packed + NB * 16 * 4 + (P + 1) * 4 + (NB + 1) * 8
    compulsory = meta_bytes + 4 * NCOL * uniq + 4 * M0 * NCOL
    gathered = meta_bytes + 4 * NCOL * sum_nact + 4 * M0 * NCOL
    achieved = compulsory / (spmm_ms / 1e3) / 1e9
    build_bytes = 8 * (M0 + 1) + 8 * nnz + packed + NB * 16 * 4 + (NB + 1) * 8 + (P + 1) * 4
    try:
        tf32_peak = measure_tf32_peak(torch)
    except Exception:
        tf32_peak = None
    exec_tflops = 2.0 * NB * args.tm * 16 * (128 * ((NCOL + 127) // 128)) / (spmm_ms / 1e3) / 1e12
    roof = {"kernel": f"hrpb::k_spmm<NT=1, TM={args.tm}>", "bound": "hbm", "achieved": round(achieved, 1), "peak": hbm,
            "unit": "GB/s", "frac": round(achieved / hbm, 4),
            "traffic": ncu_traffic(f"k_spmm_tm{args.tm}", "c2a"),
            "algorithmic_bytes_per_launch": int(compulsory),
            "bytes_definition": "packedBlocks + activeCols + blockedRowPtr + sizePtr + 4*N*(distinct columns) "
                                "+ 4*M*N (compulsory; DESIGN.md §Roofline)",
            "gathered_bytes_per_launch": int(gathered),
            "gathered_gbs": round(gathered / (spmm_ms / 1e3) / 1e9, 1),
            "kernel_ms": round(spmm_ms, 4), "share_of_step": round(spmm_ms / ms, 3),
            "peak_source": peak_src,
            "build_phase": {"ms": round(build_ms, 4),
                            "algorithmic_bytes": int(build_bytes),
                            "achieved_gbs": round(build_bytes / (build_ms / 1e3) / 1e9, 1),
                            "frac": round(build_bytes / (build_ms / 1e3) / 1e9 / hbm, 4),
                            "bytes_definition": "CSR read (8(M+1) + 8 nnz) + HRPB written (packedBlocks + "
                                                "activeCols + sizePtr + blockedRowPtr); phase = all builder "
                                                "kernels + the status read-back"},
            "tf32": {"executed_tflops": round(exec_tflops, 2),
                     "peak_tflops_measured": round(tf32_peak, 1) if tf32_peak else None,
                     "frac": round(exec_tflops / tf32_peak, 4) if tf32_peak else None}}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline_oracle(rp, ci, vals, B_h)
        except Exception as ex:  # pragma: no cover
            cpu = {"error": str(ex)}

    line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "tf32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "nnz_per_rank": nnz, "N": NCOL, "num_blocks": NB, "panels": P,
                       "bricks": bricks, "alpha": round(alpha, 4), "sum_nact": sum_nact, "distinct_cols": uniq,
                       "parallelism": f"row-panel shards x{world}, B broadcast once (NCCL)",
                       "step": "hrpb_build_spmm_async: hrpb_build (CSR->HRPB) + hrpb_spmm as one graph replay per step, no host sync between steps; every step's CSR status checked by hrpb_sync_status after the loop; build_ms/spmm_ms = library CUDA-event phase times of the last timed step and of 8 synchronous steps just before the timed region", "TM": args.tm,
                       "TK": 16,
                       "tm_plan_ms": tm_plan,
                       "l2": "inputs larger than L2 (CSR 134 MB + B 512 MB per rank)",
                       "build_ms": round(build_ms, 4), "spmm_ms": round(spmm_ms, 4),
                       "spmm_only_gflops": round(flops / (spmm_ms / 1e3) / 1e9, 1),
                       "b_broadcast_ms": round(bcast_ms, 3) if bcast_ms is not None else None},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": round(flops / (e2e_ms / 1e3) / 1e9, 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(e2e_ms, 3), "api": "hrpb_build_spmm_host (pinned host buffers)"},
            "gpu_launches": int(launches), "clocks": clk}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--tm", type=int, default=0,
                    help="HRPB panel height TM: 16 (paper default), 32, 64, or 0 = pick the fastest in an untimed plan step")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    rank, world, local_rank = env_rank()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
