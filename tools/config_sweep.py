"""All BASELINE configs on one GPU: build and SpMM times, effective GFLOP/s and the SpMM's fraction of the HBM
roofline (compulsory bytes / time / measured copy bandwidth), for each TM in a list. Writes a markdown table.

usage: python tools/config_sweep.py OUT.md [TM ...]
"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2504_06443_b200 as hp  # noqa: E402

CONFIGS = [("c1", None), ("c2a", None), ("c2b", None), ("c3", None), ("c4", None), ("c5", 32), ("c5", 128),
           ("c5", 512)]


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
    out = sys.argv[1]
    tms = [int(x) for x in sys.argv[2:]] or [16, 64]
    try:
        hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        hbm = 6650.0
    rows = ["| config | nnz | N | TM | blocks | build ms | SpMM ms | step GFLOP/s | SpMM GFLOP/s | compulsory GB | "
            "gathered GB | SpMM % of HBM (compulsory) | gathered GB/s |",
            "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    cache = {}
    for name, N in CONFIGS:
        key = name
        if key not in cache:
            cache.clear()
            cache[key] = synth.make(name)
        w0 = cache[key]
        n = N or w0.N
        dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        rp, ci, va = dev(w0.row_ptr), dev(w0.col_idx), dev(w0.vals)
        B = dev(synth.dense(w0.K, n, w0.mode, 3))
        C = torch.empty((w0.M, n), dtype=torch.float32, device="cuda")
        distinct = int(np.unique(w0.col_idx).size)
        flops = 2.0 * w0.nnz * n
        for tm in tms:
            A = hp.build(rp, ci, va, w0.M, w0.K, tm=tm)
            reps = 3 if w0.nnz > 5e7 else 10
            bms = timed(lambda: hp.build(rp, ci, va, w0.M, w0.K, tm=tm).free(), reps)
            sms = timed(lambda: hp.spmm(A, B, out=C), reps)
            _, ac, _, _ = A.to_host()
            sum_nact = int((ac < w0.K).sum())
            meta = A.packed_bytes + 4 * ac.size + 4 * (A.num_panels + 1) + 8 * (A.num_blocks + 1)
            comp = meta + 4 * n * distinct + 4 * w0.M * n
            gath = meta + 4 * n * sum_nact + 4 * w0.M * n
            line = (f"| {name} | {w0.nnz} | {n} | {tm} | {A.num_blocks} | {bms:.3f} | {sms:.3f} | "
                    f"{flops / (bms + sms) / 1e6:.0f} | {flops / sms / 1e6:.0f} | {comp / 1e9:.2f} | {gath / 1e9:.2f} | "
                    f"{100 * comp / (sms / 1e3) / 1e9 / hbm:.1f} | {gath / (sms / 1e3) / 1e9:.0f} |")
            print(line, flush=True)
            rows.append(line)
            A.free()
        del B, C, rp, ci, va
        torch.cuda.empty_cache()
    open(out, "w").write("\n".join(rows) + "\n")


if __name__ == "__main__":
    main()
