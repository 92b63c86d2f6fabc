"""Dump the activeCols of each CTA's contiguous block range (148 CTAs x NBLK blocks x 16 rows) for gather_bw /
gather_mix replay; sentinel column K is mapped to row 0.

usage: python tools/microtests/dump_rows.py OUT [TM] [WORKLOAD] [NBLK]     (defaults: 16 c2a 2048)"""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import synth
import paper_2504_06443_b200 as hp

tm = int(sys.argv[2]) if len(sys.argv) > 2 else 16
w = synth.make(sys.argv[3] if len(sys.argv) > 3 else "c2a")
d = lambda a: torch.from_numpy(a).cuda()
A = hp.build(d(w.row_ptr), d(w.col_idx), d(w.vals), w.M, w.K, tm=tm)
brp, ac, sp, _ = A.to_host()
ac = ac.reshape(-1, 16).astype(np.int64)
ac[ac == w.K] = 0
nsm, nblk = 148, int(sys.argv[4]) if len(sys.argv) > 4 else 2048
NB = ac.shape[0]
out = np.zeros((nsm, nblk, 16), np.uint32)
for c in range(nsm):
    b0 = c * NB // nsm
    blk = ac[b0:b0 + nblk]
    out[c, :blk.shape[0]] = blk
out.tofile(sys.argv[1])
print("blocks", NB, "per CTA", NB // nsm)
