"""Per-CTA wall times of one k_spmm launch of the PRODUCT kernel (HRPB_CTA_TIMES: %globaltimer at CTA entry and
exit), to measure the S1 balance without the instrumented build's distortions.

usage: python tools/cta_times.py WORKLOAD[:N] [TM]
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
path = "/tmp/hrpb_cta_times.bin"
os.environ["HRPB_CTA_TIMES"] = path
import synth  # noqa: E402
import paper_2504_06443_b200 as hp  # noqa: E402

spec = sys.argv[1]
name, N = (spec.split(":") + [None])[:2]
tm = int(sys.argv[2]) if len(sys.argv) > 2 else 16
w = synth.make(name, N=int(N) if N else None)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
A = hp.build(dev(w.row_ptr), dev(w.col_idx), dev(w.vals), w.M, w.K, tm=tm)
B = dev(w.B())
C = torch.empty((w.M, w.N), dtype=torch.float32, device="cuda")
for _ in range(3):
    hp.spmm(A, B, out=C)
torch.cuda.synchronize()
t = np.fromfile(path, dtype=np.int64).reshape(-1, 4)
t0 = t[:, 0].min()
start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
dur = end - start
print(f"{name} TM={tm} N={w.N}: kernel span {end.max():.1f} us; CTA end min/mean/max {end.min():.1f} / "
      f"{end.mean():.1f} / {end.max():.1f} us (max/mean {end.max() / end.mean():.3f}); start spread {start.max():.1f} us")
blk, pan = t[:, 2].astype(float), t[:, 3].astype(float)
print(f"  corr(dur, blocks) {np.corrcoef(dur, blk)[0, 1]:.3f}  corr(dur, panels) {np.corrcoef(dur, pan)[0, 1]:.3f}")
X = np.stack([blk, pan, np.ones_like(blk)], 1)
coef, *_ = np.linalg.lstsq(X, dur, rcond=None)
print(f"  fit us = {coef[0]:.5f} * blocks + {coef[1]:.5f} * panels + {coef[2]:.1f}  (panel/block = {coef[1] / coef[0]:.2f})")
for q in np.argsort(dur)[-4:][::-1]:
    print(f"  slow CTA {q}: {dur[q]:.0f} us, blocks {blk[q]:.0f}, panels {pan[q]:.0f}")
for q in np.argsort(dur)[:3]:
    print(f"  fast CTA {q}: {dur[q]:.0f} us, blocks {blk[q]:.0f}, panels {pan[q]:.0f}")
