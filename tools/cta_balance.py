"""Per-CTA balance of k_spmm (S1): cycles, blocks, panels per CTA from an instrumented build.

usage: python tools/build_variant.py instr -DHRPB_INSTRUMENT=1
       python tools/cta_balance.py .variants/instr.so WORKLOAD [TM]
Prints max/mean cycles and how per-CTA cycles correlate with its blocks, panels and position.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
import paper_2504_06443_b200 as hp  # noqa: E402

hp.hrpb._SO = os.path.abspath(sys.argv[1])
name = sys.argv[2]
tm = int(sys.argv[3]) if len(sys.argv) > 3 else 16
path = "/tmp/hrpb_trace.bin"
os.environ["HRPB_TRACE"] = path
w = synth.make(name)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
A = hp.build(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), w.M, w.K, tm=tm)
B = dev(w.B())
C = torch.empty((w.M, w.N), dtype=torch.float32, device="cuda")
hp.spmm(A, B, out=C)
torch.cuda.synchronize()
hp.spmm(A, B, out=C)
torch.cuda.synchronize()
t = np.fromfile(path, dtype=np.int64).reshape(10, 1024)[9].reshape(256, 4)
G = torch.cuda.get_device_properties(0).multi_processor_count
t = t[:G]
cyc, blk, pan, pa = t[:, 0].astype(float), t[:, 1].astype(float), t[:, 2].astype(float), t[:, 3]
print(f"{name} TM={tm} N={w.N}: CTA cycles max/mean {cyc.max() / cyc.mean():.3f} (min/mean {cyc.min() / cyc.mean():.3f})")
print(f"  blocks per CTA mean {blk.mean():.0f} [{blk.min():.0f}, {blk.max():.0f}], panels [{pan.min():.0f}, {pan.max():.0f}]")
print(f"  corr(cycles, blocks) {np.corrcoef(cyc, blk)[0, 1]:.3f}  corr(cycles, panels) {np.corrcoef(cyc, pan)[0, 1]:.3f}"
      f"  corr(cycles, position) {np.corrcoef(cyc, np.arange(G))[0, 1]:.3f}")
# least squares: cycles ~ a * blocks + b * panels + c
X = np.stack([blk, pan, np.ones_like(blk)], 1)
coef, *_ = np.linalg.lstsq(X, cyc, rcond=None)
print(f"  fit cycles = {coef[0]:.0f} * blocks + {coef[1]:.0f} * panels + {coef[2]:.0f}")
for q in np.argsort(cyc)[-5:][::-1]:
    print(f"  slow CTA {q}: cycles {cyc[q]:.3g} blocks {blk[q]:.0f} panels {pan[q]:.0f} first panel {pa[q]}")
for q in np.argsort(cyc)[:3]:
    print(f"  fast CTA {q}: cycles {cyc[q]:.3g} blocks {blk[q]:.0f} panels {pan[q]:.0f} first panel {pa[q]}")
