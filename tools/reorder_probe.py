"""NEXT-4 probe: reorder cost and its effect on the HRPB (blocks, sum nact, alpha) and on build / SpMM time.

usage: python tools/reorder_probe.py WORKLOAD[:N] [TM]
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


spec = sys.argv[1]
name, N = (spec.split(":") + [None])[:2]
tm = int(sys.argv[2]) if len(sys.argv) > 2 else 16
w = synth.make(name, N=int(N) if N else None)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
rp, ci, va = dev(w.row_ptr), dev(w.col_idx), dev(w.vals)
B = dev(w.B())
C = torch.empty((w.M, w.N), dtype=torch.float32, device="cuda")
flops = 2.0 * w.nnz * w.N
rms = timed(lambda: hp.reorder_rows(rp, ci, va, w.M, w.K), 5)
perm, rp2, ci2, v2 = hp.reorder_rows(rp, ci, va, w.M, w.K)
for label, (r, c, v, pm) in (("original", (rp, ci, va, None)), ("reordered", (rp2, ci2, v2, perm))):
    A = hp.build(r, c, v, w.M, w.K, tm=tm)
    if pm is not None:
        A.set_row_map(pm)
    bms = timed(lambda: hp.build(r, c, v, w.M, w.K, tm=tm).free(), 3)
    sms = timed(lambda: hp.spmm(A, B, out=C), 5)
    _, ac, _, _ = A.to_host()
    extra = f"  reorder {rms:.3f} ms" if pm is not None else ""
    print(f"{name} N={w.N} TM={tm} {label:9s}: blocks {A.num_blocks}  sum_nact {int((ac < w.K).sum())}  "
          f"build {bms:.3f} ms  spmm {sms:.3f} ms ({flops / sms / 1e6:.0f} GF/s){extra}", flush=True)
    A.free()
