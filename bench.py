#!/usr/bin/env python
"""bench.py — HRPB SpMM on B200 (the hot path of cuTeSpMM, arxiv 2504.06443).

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c3] [--tm 0]
                [--weight nnz|nact] [--no-per-config] [--no-cpu-baseline]

One step = one pass of the whole hot path over one synthetic matrix: hrpb_build (CSR -> HRPB on the GPU,
SURVEY §8(a) B1-B5) + hrpb_spmm (S1-S5), inputs resident in HBM, enqueued by one hrpb_build_spmm_async call
(graph-replayed; every step's CSR status is checked by hrpb_sync_status after the loop).

Workload ("c3 is the headline number"): BASELINE configs[2], R-MAT scale 22 (M = K = 4,194,304,
edge factor 32, Graph500 (0.57, 0.19, 0.19, 0.05), duplicates removed: 128.3M nnz), N = 256, float mode, TM chosen
by the library (tm = 0). With N GPUs (one process per GPU, self-spawned through torch.distributed.run when
WORLD_SIZE is unset) the row panels are partitioned by dist.shard_plan (contiguous ranges of equal nnz — the north
star — or equal HRPB blocks with --weight nact), B is broadcast once over NCCL (timed separately) and every rank
writes its own C rows: strong scaling, no reduction.

At N = 1 the same JSON line carries `per_config`: c1, c2a, c2b, c4 and c5 @ N = 32/128/512, each with its build and
SpMM times and the SpMM's roofline under three byte counts side by side.

Metric: effective GFLOP/s = 2 * nnz * N / t (BASELINE.json metric), whole job.
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "SpMM effective GFLOP/s (2*nnz*N/t) and % HBM/TF32 roofline"
UNIT = "GFLOP/s"
WORKLOADS = {
    "c3": "c3: R-MAT scale 22 (M=K=4,194,304, edge factor 32, (0.57,0.19,0.19,0.05), duplicates removed), N=256, "
          "float mode (BASELINE configs[2]; SURVEY §8(d) headline)",
    "c2a": "c2a: banded M=K=2^20, 16 distinct nnz/row uniform in [i-32,i+32), N=128, float mode (BASELINE configs[1])",
    "c2b": "c2b: block-clustered M=K=2^20, 4 dense 16x4 clusters per 16-row panel, N=128, float (BASELINE configs[1])",
    "c4": "c4: uniform M=K=2^21, 8 distinct nnz/row, N=512, float mode (BASELINE configs[3])",
    "c5": "c5: FEM 250x250 nodes x 8 dofs (M=K=500,000), dense 8x8 blocks on a 9-point stencil + 1 random block "
          "per block row, float mode (BASELINE configs[4])",
    "c1": "c1: uniform random M=K=4096, Bernoulli(0.01), N=32, exact mode (BASELINE configs[0])",
}
PER_CONFIG = [("c1", None), ("c2a", None), ("c2b", None), ("c4", None), ("c5", 32), ("c5", 128), ("c5", 512)]


def env_rank():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), \
        int(os.environ.get("LOCAL_RANK", "0"))


def free_port():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def read_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


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
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.2)
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


def ncu_traffic(tag: str, kernel: str):
    """DRAM bytes (read + write) per launch of `kernel` on workload `tag` from the committed ncu --set full
    summaries (profiles/ncu_traffic.json, written by tools/ncu_summary.py)."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_traffic.json")))
        return d.get(tag, {}).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
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


# ------------------------------------------------------------------------------------------ workloads
def shared_dir():
    return f"/dev/shm/hrpb_bench_{os.environ.get('MASTER_PORT', os.getpid())}"


def load_full(name, N=None):
    """The whole synthetic matrix (host arrays): generated once per node — rank 0 generates and shares it
    through /dev/shm when several ranks run (the R-MAT generator is global over edges)."""
    rank, world, _ = env_rank()
    if world == 1:
        return synth.make(name, N=N)
    import torch.distributed as dist
    d = shared_dir()
    if rank == 0:
        w = synth.make(name, N=N)
        os.makedirs(d, exist_ok=True)
        for k in ("row_ptr", "col_idx", "vals"):
            np.save(os.path.join(d, k + ".npy"), getattr(w, k))
        json.dump({"name": w.name, "M": w.M, "K": w.K, "N": w.N, "mode": w.mode}, open(os.path.join(d, "meta.json"), "w"))
    dist.barrier()
    if rank != 0:
        m = json.load(open(os.path.join(d, "meta.json")))
        arr = {k: np.load(os.path.join(d, k + ".npy"), mmap_mode="r") for k in ("row_ptr", "col_idx", "vals")}
        w = synth.Workload(m["name"], m["M"], m["K"], m["N"], m["mode"], arr["row_ptr"], arr["col_idx"], arr["vals"])
    dist.barrier()
    if rank == 0:
        for k in ("row_ptr", "col_idx", "vals"):
            os.unlink(os.path.join(d, k + ".npy"))
    return w


def roof_bytes(A_stats, N, M, distinct, sum_nact):
    """The SpMM's bytes per launch under the two model definitions: 'gathered' = the algorithmic
    bytes_alg (packedBlocks + activeCols + blockedRowPtr + sizePtr + 4 N sum_p nact(p) + 4 M N) and 'compulsory'
    (each distinct B row once: 4 N |distinct columns| instead of the gathered term)."""
    packed, NB, P, tk = A_stats
    meta = packed + 4 * tk * NB + 4 * (P + 1) + 8 * (NB + 1)
    return meta + 4 * N * sum_nact + 4 * M * N, meta + 4 * N * distinct + 4 * M * N


def hrpb_stats(hp, rp_d, ci_d, v_d, M, K, tm, tk=16):
    """Structure of the HRPB the step builds (outside the timed region): sizes, sum of nact, bricks, alpha."""
    A = hp.build(rp_d, ci_d, v_d, M, K, tm=tm, tk=tk)
    brp, ac, sp, packed_h = A.to_host()
    out = {"tm": A.tm, "num_blocks": A.num_blocks, "panels": A.num_panels, "packed_bytes": A.packed_bytes,
           "sum_nact": int(np.count_nonzero(ac != K))}
    nbr = packed_h[sp[:-1].astype(np.int64) + tk // 4].astype(np.int64) if A.num_blocks else np.zeros(0, np.int64)
    out["bricks"] = int(nbr.sum())
    out["alpha"] = round(int(A.nnz) / max(1, 64 * out["bricks"]), 4)  # brick density
    out["blocks_per_panel"] = np.diff(brp.astype(np.int64))
    A.free()
    return out


# ------------------------------------------------------------------------------------------ reference arm
def run_reference(args, rank, world):
    """The tier's reference arm: the CPU oracle as it stands, on this box's host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle
    w = synth.make(args.workload)
    B = w.B()
    M, K, N = w.M, w.K, w.N
    total_steps = args.steps + args.warmup
    budget = 150.0  # seconds for the whole run
    # one reference step = oracle CSR->HRPB conversion + oracle CSR SpMM on a row sample (mirrors build + SpMM)
    probe_rows = 16 * 256
    t = time.perf_counter()
    oracle.csr_to_hrpb(M, K, w.row_ptr, w.col_idx, w.vals, p0=0, p1=probe_rows // 16)
    oracle.csr_spmm_f32out(M, w.row_ptr, w.col_idx, w.vals, B, 0, probe_rows)
    per_row = (time.perf_counter() - t) / probe_rows
    rows = int(max(16, min(M, budget / total_steps / max(per_row, 1e-12))) // 16 * 16)
    out = np.empty((rows, N), np.float32)
    th = oracle.num_threads()

    def step():
        oracle.csr_to_hrpb(M, K, w.row_ptr, w.col_idx, w.vals, p0=0, p1=rows // 16)
        oracle.csr_spmm_f32out(M, w.row_ptr, w.col_idx, w.vals, B, 0, rows, out=out)

    for _ in range(args.warmup):
        step()
    t = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t) / max(args.steps, 1)
    nnz_s = int(w.row_ptr[rows])
    v = 2.0 * nnz_s * N / dt / 1e9
    sample = (f"rows [0,{rows}) of {args.workload} ({nnz_s} nnz) per step: oracle CSR->HRPB (serial) + "
              f"oracle CSR SpMM (FP64 acc, OpenMP)")
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS[args.workload], "sample_rows": rows},
            "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": th, "kind": "oracle", "sample": sample,
                             "nproc": os.cpu_count(), "cpu_model": cpu_model()},
            "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_oracle(w, B, target_s=12.0, cap_s=30.0):
    """Oracle CSR SpMM (FP64 accumulate, fp32 out, OpenMP over rows) on the host cores; bounded sample: a row
    prefix sized from a probe so that one pass is <= target_s, repeated until ~target_s of CPU work (cap cap_s)."""
    import oracle
    M = w.M
    probe = min(M, 65536)
    t = time.perf_counter()
    oracle.csr_spmm_f32out(M, w.row_ptr, w.col_idx, w.vals, B, 0, probe)
    per_nnz = (time.perf_counter() - t) / max(1, int(w.row_ptr[probe]))
    rows = M
    if per_nnz * w.nnz > target_s:  # rows of the prefix holding ~target_s of work
        rows = int(np.searchsorted(w.row_ptr, target_s / per_nnz)) or probe
    out = np.empty((rows, B.shape[1]), np.float32)
    reps, th = 0, 1
    t = time.perf_counter()
    while True:
        _, th = oracle.csr_spmm_f32out(M, w.row_ptr, w.col_idx, w.vals, B, 0, rows, out=out)
        reps += 1
        dt = time.perf_counter() - t
        if dt >= target_s or dt * (reps + 1) / reps > cap_s:
            break
    nnz_s = int(w.row_ptr[rows] - w.row_ptr[0])
    gf = 2.0 * nnz_s * B.shape[1] * reps / dt / 1e9
    return {"value": round(gf, 3), "unit": UNIT, "cores": int(th), "kind": "oracle",
            "nproc": os.cpu_count(), "cpu_model": cpu_model(),
            "affinity": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
            "sample": f"rows [0,{rows}) of {w.name} ({nnz_s} nnz of {w.nnz}), N={B.shape[1]}, x{reps}, {dt:.1f} s, "
                      f"FP64-accumulating CSR SpMM with fp32 output (oracle/oracle.c)"}


# ------------------------------------------------------------------------------------------ our arm
class Stepper:
    """Times the hot path (hrpb_build_spmm_async, graph-replayed) on one matrix resident in HBM."""

    def __init__(self, torch, hp, rp, ci, vals, B_d, M, K, tm, stream):
        self.torch, self.hp, self.stream = torch, hp, stream
        dev = B_d.device
        self.rp = torch.from_numpy(np.ascontiguousarray(rp)).to(dev)
        self.ci = torch.from_numpy(np.ascontiguousarray(ci)).to(dev)
        self.v = torch.from_numpy(np.ascontiguousarray(vals)).to(dev)
        self.B, self.M, self.K, self.tm = B_d, M, K, tm
        self.C = torch.empty((M, B_d.shape[1]), dtype=torch.float32, device=dev)
        self.nnz = int(ci.shape[0])

    def sync_step(self):
        _, _, ms = self.hp.build_spmm(self.rp, self.ci, self.v, self.B, self.M, self.K, out=self.C, tm=self.tm,
                                      stream=self.stream)
        return ms

    def async_step(self):
        self.hp.build_spmm_async(self.rp, self.ci, self.v, self.B, self.M, self.K, self.C, tm=self.tm,
                                 stream=self.stream)

    def warm(self, warmup, phase_steps=5):
        for _ in range(max(warmup, 3)):
            self.sync_step()
        phases = [self.sync_step() for _ in range(phase_steps)]
        self.async_step()
        self.hp.sync_status(self.stream)
        self.torch.cuda.synchronize()
        return phases

    def timed(self, steps):
        torch = self.torch
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(self.stream)
        for _ in range(steps):
            self.async_step()
        t1.record(self.stream)
        last = self.hp.sync_status(self.stream)  # raises if any timed step saw an invalid CSR
        torch.cuda.synchronize()
        return t0.elapsed_time(t1) / max(steps, 1), last


def measure_config(torch, hp, name, N, stream, hbm, steps=10):
    """One per_config record: build + SpMM step time, phase times, and the SpMM's roofline."""
    w = synth.make(name, N=N)
    B_d = torch.from_numpy(w.B()).cuda()
    st = Stepper(torch, hp, w.row_ptr, w.col_idx, w.vals, B_d, w.M, w.K, 0, stream)
    phases = st.warm(3)
    ms, last = st.timed(steps)
    phases.append(last)
    build_ms = float(np.median([p[0] for p in phases]))
    spmm_ms = float(np.median([p[1] for p in phases]))
    hs = hrpb_stats(hp, st.rp, st.ci, st.v, w.M, w.K, 0)
    distinct = int(np.count_nonzero(np.bincount(w.col_idx, minlength=w.K)))
    gathered, compulsory = roof_bytes((hs["packed_bytes"], hs["num_blocks"], hs["panels"], 16), w.N, w.M, distinct,
                                      hs["sum_nact"])
    flops = 2.0 * w.nnz * w.N
    tag = f"{name}_N{w.N}_tm{hs['tm']}"
    traffic = ncu_traffic(tag, "k_spmm")
    rec = {"workload": WORKLOADS[name] if N is None else WORKLOADS[name] + f", N={w.N}",
           "nnz": w.nnz, "N": w.N, "TM": hs["tm"], "num_blocks": hs["num_blocks"], "alpha": hs["alpha"],
           "ms_per_step": round(ms, 4), "value": round(flops / (ms / 1e3) / 1e9, 1),
           "build_ms": round(build_ms, 4), "spmm_ms": round(spmm_ms, 4),
           "spmm_only_gflops": round(flops / (spmm_ms / 1e3) / 1e9, 1),
           "spmm_roofline": {
               "peak_gbs": hbm,
               "gathered_bytes": int(gathered), "gathered_frac": round(gathered / (spmm_ms / 1e3) / 1e9 / hbm, 4),
               "compulsory_bytes": int(compulsory),
               "compulsory_frac": round(compulsory / (spmm_ms / 1e3) / 1e9 / hbm, 4),
               "ncu_dram_bytes": traffic,
               "ncu_dram_frac": round(traffic / (spmm_ms / 1e3) / 1e9 / hbm, 4) if traffic else None}}
    del st, B_d
    torch.cuda.empty_cache()
    return rec


def run_ours(args, rank, world, local_rank):
    import torch
    import paper_2504_06443_b200 as hp
    from paper_2504_06443_b200 import dist as hdist
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream()  # non-default: the library graph-captures the repeated step
    torch.cuda.set_stream(stream)

    w = load_full(args.workload)
    M, K, N = w.M, w.K, w.N
    # ---------------------------------------------------------------- partition (N > 1) and B broadcast
    shard = None
    if world > 1:
        weights = None
        if args.weight == "nact":  # blocks per panel from one GPU build of the whole matrix (B1 counts, rank 0)
            cnt = torch.zeros(((M + 15) // 16,), dtype=torch.int64, device=dev)
            if rank == 0:
                g = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
                A = hp.build(g(w.row_ptr), g(w.col_idx), g(w.vals), M, K, tm=16)
                brp = A.to_host()[0].astype(np.int64)
                A.free()
                cnt.copy_(torch.from_numpy(np.diff(brp)))
            dist.broadcast(cnt, src=0)
            weights = cnt.cpu().numpy()
        shard = hdist.shard_plan(w.row_ptr, world, 16, args.weight if weights is None else weights)[rank]
        rp, ci, vals = hdist.slice_rows(w.row_ptr, w.col_idx, w.vals, shard)
        Ml = shard.nrows
    else:
        rp, ci, vals, Ml = w.row_ptr, w.col_idx, w.vals, M
    B_h = w.B() if rank == 0 else None
    B_d = torch.from_numpy(B_h).to(dev) if rank == 0 else torch.empty((K, N), dtype=torch.float32, device=dev)
    bcast_ms = None
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        hdist.broadcast_B(B_d)  # the path's only collective (ncclBroadcast over NVLink / NVSwitch)
        e.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([s.elapsed_time(e)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        bcast_ms = float(t[0])

    st = Stepper(torch, hp, rp, ci, vals, B_d, Ml, K, args.tm, stream)
    nnz_local = st.nnz
    phases = st.warm(args.warmup, 8)
    hs = hrpb_stats(hp, st.rp, st.ci, st.v, Ml, K, args.tm)  # (outside the timed region)
    tm = hs["tm"]
    distinct = int(np.count_nonzero(np.bincount(np.asarray(ci), minlength=K)))

    # ---------------------------------------------------------------- timed region
    clocks = ClockSampler(local_rank)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = hp.launch_count()
    ms, last_phase = st.timed(args.steps)
    if world > 1:
        dist.barrier()
    launches = hp.launch_count() - launches0
    clk = clocks.stop()
    phases.append(last_phase)
    build_ms = float(np.median([p[0] for p in phases]))
    spmm_ms = float(np.median([p[1] for p in phases]))
    stats = torch.tensor([ms, build_ms, spmm_ms, float(nnz_local), float(launches)], dtype=torch.float64, device=dev)
    if world > 1:
        mx = stats.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = stats.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, build_ms, spmm_ms = float(mx[0]), float(mx[1]), float(mx[2])
        total_nnz, launches = float(sm[3]), int(sm[4])
    else:
        total_nnz = float(nnz_local)
    flops = 2.0 * total_nnz * N
    value = flops / (ms / 1e3) / 1e9

    # ---------------------------------------------------------------- e2e through the host C-ABI entry point
    if B_h is None:
        B_h = B_d.cpu().numpy()
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    rp_h, ci_h, v_h, Bp_h = pin(rp), pin(ci), pin(vals), pin(B_h)
    Cp_h = torch.empty((Ml, N), dtype=torch.float32).pin_memory()
    hp.build_spmm_host(rp_h, ci_h, v_h, Bp_h, Ml, K, out=Cp_h, tm=tm)  # warm
    e2e_steps = max(1, min(args.steps, 3))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(e2e_steps):
        hp.build_spmm_host(rp_h, ci_h, v_h, Bp_h, Ml, K, out=Cp_h, tm=tm)
    e.record(stream)
    torch.cuda.synchronize()
    e2e_ms = s.elapsed_time(e) / e2e_steps
    io = torch.tensor([e2e_ms, (Ml + 1) * 8 + nnz_local * 8 + K * N * 4, Ml * N * 4], dtype=torch.float64, device=dev)
    if world > 1:
        mx = io.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = io.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        e2e_ms, h2d, d2h = float(mx[0]), int(sm[1]), int(sm[2])
    else:
        h2d, d2h = int(io[1]), int(io[2])
    del rp_h, ci_h, v_h, Bp_h, Cp_h

    # ---------------------------------------------------------------- roofline of the dominant kernel
    peaks = read_peaks()
    hbm = peaks.get("hbm_gbs")
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured copy bandwidth)"
    if not hbm:
        hbm, peak_src = 6650.0, "fallback 6.65 TB/s (B200_PROFILING.md)"
    gathered, compulsory = roof_bytes((hs["packed_bytes"], hs["num_blocks"], hs["panels"], 16), N, Ml, distinct,
                                      hs["sum_nact"])
    build_bytes = 8 * (Ml + 1) + 8 * nnz_local + hs["packed_bytes"] + hs["num_blocks"] * 16 * 4 + \
        (hs["num_blocks"] + 1) * 8 + (hs["panels"] + 1) * 4
    tag = f"{args.workload}_N{N}_tm{tm}" + (f"_r{rank}of{world}" if world > 1 else "")
    traffic = ncu_traffic(tag, "k_spmm")
    spmm_dominant = spmm_ms >= build_ms

    per_config = None
    tf32_peak = None
    cpu = None
    if rank == 0 and world == 1:
        try:
            tf32_peak = measure_tf32_peak(torch)
        except Exception:
            tf32_peak = None
        if not args.no_per_config:
            del st
            torch.cuda.empty_cache()
            per_config = {}
            for name, n in PER_CONFIG:
                key = name if n is None else f"{name}@N{n}"
                try:
                    per_config[key] = measure_config(torch, hp, name, n, stream, hbm)
                except Exception as ex:  # pragma: no cover
                    per_config[key] = {"error": repr(ex)}
        if not args.no_cpu_baseline:
            try:
                cpu = cpu_baseline_oracle(w, B_h)
            except Exception as ex:  # pragma: no cover
                cpu = {"error": str(ex)}

    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return

    in_bytes = 8 * (Ml + 1) + 8 * nnz_local + 4 * K * N
    l2_note = ("inputs larger than L2 (CSR + B > 2 x 126 MB): no flush between steps" if in_bytes > 2 * 126e6 else
               "inputs fit L2: no flush between steps (steady-state repeated SpMM, P:L484)")
    exec_tflops = 2.0 * hs["num_blocks"] * tm * 16 * (128 * ((N + 127) // 128)) / (spmm_ms / 1e3) / 1e12
    roof = {"kernel": f"hrpb::k_spmm<NT={min(4, (N + 127) // 128)}, TM={tm}>" if spmm_dominant else "hrpb builder",
            "bound": "hbm", "unit": "GB/s", "peak": hbm, "peak_source": peak_src,
            "achieved": round(gathered / (spmm_ms / 1e3) / 1e9, 1),
            "frac": round(gathered / (spmm_ms / 1e3) / 1e9 / hbm, 4),
            "frac_definition": "gathered: SURVEY §8(d) bytes_alg = packedBlocks + activeCols + blockedRowPtr + "
                               "sizePtr + 4*N*sum_p nact(p) + 4*M*N per launch / kernel time / peak (> 1 means L2 "
                               "served re-gathered B rows)",
            "traffic": traffic,
            "algorithmic_bytes_per_launch": int(gathered),
            "compulsory_bytes_per_launch": int(compulsory),
            "compulsory_frac": round(compulsory / (spmm_ms / 1e3) / 1e9 / hbm, 4),
            "ncu_dram_frac": round(traffic / (spmm_ms / 1e3) / 1e9 / hbm, 4) if traffic else None,
            "kernel_ms": round(spmm_ms, 4), "share_of_step": round(spmm_ms / ms, 3),
            "build_phase": {"ms": round(build_ms, 4), "algorithmic_bytes": int(build_bytes),
                            "achieved_gbs": round(build_bytes / (build_ms / 1e3) / 1e9, 1),
                            "frac": round(build_bytes / (build_ms / 1e3) / 1e9 / hbm, 4),
                            "share_of_step": round(build_ms / ms, 3),
                            "bytes_definition": "CSR read (8(M+1) + 8 nnz) + HRPB written (packedBlocks + activeCols "
                                                "+ sizePtr + blockedRowPtr); phase = every builder kernel + read-back"},
            "tf32": {"executed_tflops": round(exec_tflops, 2),
                     "peak_tflops_measured": round(tf32_peak, 1) if tf32_peak else None,
                     "frac": round(exec_tflops / tf32_peak, 4) if tf32_peak else None}}
    if world > 1:
        roof["note"] = "rank 0's SpMM; times are the max over ranks"
    line = {"metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "tf32",
            "data": "synthetic (seeded generators, synth/)",
            "config": {"workload": WORKLOADS[args.workload], "nnz": int(total_nnz), "N": N, "M": M, "K": K,
                       "TM": tm, "TK": 16, "TM_choice": "library (hrpb_config_t.tm = 0)" if args.tm == 0 else "fixed",
                       "num_blocks_rank0": hs["num_blocks"], "panels_rank0": hs["panels"],
                       "bricks_rank0": hs["bricks"], "alpha": hs["alpha"], "sum_nact_rank0": hs["sum_nact"],
                       "distinct_cols_rank0": distinct,
                       "parallelism": (f"row panels sharded over {world} ranks by dist.shard_plan (weight "
                                       f"{args.weight}), B broadcast once (NCCL), no reduction") if world > 1
                       else "1 GPU",
                       "step": "hrpb_build_spmm_async: hrpb_build (CSR->HRPB) + hrpb_spmm as one graph replay, no "
                               "host sync between steps; every step's CSR status checked by hrpb_sync_status after "
                               "the loop; build_ms/spmm_ms = median of the library's CUDA-event phase times (8 "
                               "synchronous steps before + the last timed step)",
                       "l2": l2_note, "input_bytes_rank0": int(in_bytes),
                       "build_ms": round(build_ms, 4), "spmm_ms": round(spmm_ms, 4),
                       "spmm_only_gflops": round(flops / (spmm_ms / 1e3) / 1e9, 1),
                       "b_broadcast_ms": round(bcast_ms, 3) if bcast_ms is not None else None,
                       "shard_rank0": None if shard is None else {"p0": shard.p0, "p1": shard.p1,
                                                                 "nnz": nnz_local}},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": round(flops / (e2e_ms / 1e3) / 1e9, 2), "unit": UNIT,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": round(e2e_ms, 3),
                    "api": "hrpb_build_spmm_host (pinned host buffers: CSR + B in, C out, inside the timed region)"},
            "gpu_launches": int(launches), "clocks": clk, "per_config": per_config}
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


# ------------------------------------------------------------------------------------------ orchestration check
def run_cpu_check(args, rank, world):
    """--cpu-check (tests only): the multi-rank orchestration on CPU with gloo — the same partition, B broadcast,
    max-over-ranks and JSON line — with each rank's rows computed by the CPU oracle instead of the CUDA library.
    Exercises the self-spawn path without a GPU; never used for a measurement."""
    import torch
    import torch.distributed as dist
    import oracle
    from paper_2504_06443_b200 import dist as hdist
    if world > 1:
        dist.init_process_group("gloo")
    w = synth.make(args.workload, scale=9, N=8)
    shard = hdist.shard_plan(w.row_ptr, world, 16, args.weight if args.weight != "nact" else "nnz")[rank]
    rp, ci, vals = hdist.slice_rows(w.row_ptr, w.col_idx, w.vals, shard)
    B = torch.from_numpy(w.B()) if rank == 0 else torch.zeros((w.K, w.N), dtype=torch.float32)
    if world > 1:
        hdist.broadcast_B(B)
    t = time.perf_counter()
    C = oracle.csr_spmm(shard.nrows, w.K, rp, ci, vals, B.numpy())
    dt = time.perf_counter() - t
    full = oracle.csr_spmm(w.M, w.K, w.row_ptr, w.col_idx, w.vals, w.B())
    ok = np.array_equal(C, full[shard.row0:shard.row0 + shard.nrows])
    st = torch.tensor([dt, float(ci.shape[0]), float(shard.nrows), float(ok)], dtype=torch.float64)
    if world > 1:
        mx = st.clone(); dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = st.clone(); dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        mn = st.clone(); dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        dt, nnz, rows, ok = float(mx[0]), int(sm[1]), int(sm[2]), bool(mn[3])
    else:
        nnz, rows = int(ci.shape[0]), shard.nrows
    if rank == 0:
        print(json.dumps({"impl": "cpu-check", "n_gpus": world, "world": world, "rows": rows, "M": w.M, "nnz": nnz,
                          "total_nnz": w.nnz, "parity": ok, "ms": round(dt * 1e3, 3),
                          "scaling": "strong"}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--tm", type=int, default=0, help="HRPB panel height: 0 = the library's choice (default)")
    ap.add_argument("--weight", default="nnz", choices=["nnz", "nact"],
                    help="N > 1 partition weight: nnz per panel (north star) or HRPB blocks per panel (B1 counts)")
    ap.add_argument("--no-per-config", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-check", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch through torch.distributed.run (the driver's own launch form)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    rank, world, local_rank = env_rank()
    if args.gpus != world and not args.cpu_check:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
    if args.cpu_check:
        run_cpu_check(args, rank, world)
    elif args.impl == "reference":
        args.warmup = max(args.warmup, 1)
        run_reference(args, rank, world)
    else:
        args.warmup = max(args.warmup, 3)
        run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
