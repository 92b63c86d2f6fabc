"""Per-config timing probe (diagnostics, not the bench): build + spmm on one synthetic workload.

usage: python tools/spmm_probe.py [--lib PATH.so] WORKLOAD[:N] [TM ...]   e.g.  c2a 16 32 64   c5:512 16 64

Prints one line per (workload, TM): build ms, spmm ms, effective GFLOP/s, gathered GB/s (4*N*sum_nact +
A + C bytes over the SpMM time) and compulsory GB/s (distinct B rows instead of the gathered ones).
Environment knobs of the library (HRPB_DEBUG, HRPB_GATHER) apply as usual.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2504_06443_b200 as hp  # noqa: E402


def timed(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


def main():
    if sys.argv[1] == "--lib":  # experimental variant built by tools/build_variant.py
        hp.hrpb._SO = os.path.abspath(sys.argv[2])
        del sys.argv[1:3]
    spec = sys.argv[1]
    name, N = (spec.split(":") + [None])[:2]
    # TM or TMxTK (e.g. 64x32)
    tms = [tuple(int(y) for y in x.split("x")) if "x" in x else (int(x), 16) for x in sys.argv[2:]] or [(16, 16)]
    w = synth.make(name, N=int(N) if N else None)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    rp, ci, va = dev(w.row_ptr), dev(w.col_idx), dev(w.vals)
    B = dev(w.B())
    C = torch.empty((w.M, w.N), dtype=torch.float32, device="cuda")
    flops = 2.0 * w.nnz * w.N
    distinct = int(np.unique(w.col_idx).size)
    for tm, tk in tms:
        A = hp.build(rp, ci, va, w.M, w.K, tm=tm, tk=tk)
        bms = timed(lambda: hp.build(rp, ci, va, w.M, w.K, tm=tm, tk=tk).free(), 5)
        sms = timed(lambda: hp.spmm(A, B, out=C), 10)
        _, ac, _, _ = A.to_host()
        sum_nact = int((ac < w.K).sum())
        meta = A.packed_bytes + 4 * ac.size + 4 * (A.num_panels + 1) + 8 * (A.num_blocks + 1)
        gath = meta + 4 * w.N * sum_nact + 4 * w.M * w.N
        comp = meta + 4 * w.N * distinct + 4 * w.M * w.N
        print(f"{name} N={w.N} nnz={w.nnz} TM={tm} TK={tk} NB={A.num_blocks} build {bms:.3f} ms  spmm {sms:.3f} ms  "
              f"{flops / sms / 1e6:.0f} GF/s spmm-only, {flops / (sms + bms) / 1e6:.0f} GF/s step  "
              f"gathered {gath / sms / 1e6:.0f} GB/s  compulsory {comp / sms / 1e6:.0f} GB/s", flush=True)
        A.free()


if __name__ == "__main__":
    main()
