"""Times the end-to-end host entry point (hrpb_build_spmm_host) on c2a from pinned host buffers.

usage: python tools/e2e_probe.py [--lib PATH.so] [TM]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2504_06443_b200 as hp  # noqa: E402

if len(sys.argv) > 2 and sys.argv[1] == "--lib":
    hp.hrpb._SO = os.path.abspath(sys.argv[2])
    del sys.argv[1:3]
tm = int(sys.argv[1]) if len(sys.argv) > 1 else 64
w = synth.make("c2a")
pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
rp, ci, va, B = pin(w.row_ptr), pin(w.col_idx), pin(w.vals), pin(w.B())
C = torch.empty((w.M, w.N), dtype=torch.float32).pin_memory()
hp.build_spmm_host(rp, ci, va, B, w.M, w.K, out=C, tm=tm)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    hp.build_spmm_host(rp, ci, va, B, w.M, w.K, out=C, tm=tm)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 5
print(f"e2e c2a TM={tm}: {ms:.3f} ms  ({2 * w.nnz * w.N / ms / 1e6:.1f} GFLOP/s)")
# PCIe floor: the same bytes with plain copies — serial, and H2D || D2H on two streams
dB = torch.empty_like(B, device="cuda"); dci = torch.empty_like(ci, device="cuda"); dva = torch.empty_like(va, device="cuda")
drp = torch.empty_like(rp, device="cuda"); dC = torch.empty_like(C, device="cuda")
s2 = torch.cuda.Stream()
for mode in ("serial", "overlap"):
    torch.cuda.synchronize()
    s.record()
    for _ in range(3):
        for src, dst in ((rp, drp), (ci, dci), (va, dva), (B, dB)):
            dst.copy_(src, non_blocking=True)
        if mode == "overlap":
            with torch.cuda.stream(s2):
                C.copy_(dC, non_blocking=True)
        else:
            C.copy_(dC, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
    e.record()
    torch.cuda.synchronize()
    print(f"copies only ({mode}): {s.elapsed_time(e) / 3:.3f} ms")
