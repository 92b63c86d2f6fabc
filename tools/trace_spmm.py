"""Analyse an HRPB_TRACE dump (CTA 0 per-block clock64 events of k_spmm)."""
import sys
import numpy as np

N = 1024
raw = np.fromfile(sys.argv[1], dtype=np.int64)
t = raw.reshape(raw.size // N, N).astype(np.float64)
valid = (t[0] > 0) & (t[4] > 0)
n = int(valid.sum())
t0 = t[0][valid].min()
names = ["issue", "a_ready", "dec_done", "b_ready", "mma", "tfull", "dec_table", "dec_rows"][:t.shape[0]]
ev = {k: t[i][:n] - t0 for i, k in enumerate(names)}
print(f"blocks traced: {n}")
for a, b in [("issue", "a_ready"), ("a_ready", "dec_table"), ("dec_table", "dec_rows"), ("dec_rows", "dec_done"), ("a_ready", "dec_done"), ("issue", "b_ready"), ("dec_done", "mma"),
             ("b_ready", "mma"), ("issue", "mma")]:
    d = ev[b] - ev[a]
    print(f"{a:>9s} -> {b:<9s}: median {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f} cycles")
iss = np.diff(ev["issue"])
print(f"issue interval median {np.median(iss):.0f} cycles; mma interval median {np.median(np.diff(ev['mma'])):.0f}")
start = int(sys.argv[2]) if len(sys.argv) > 2 else 0
print(f"blocks {start}..{start + 24} (cycles rel. to first issue):")
for i in range(start, min(start + 24, n)):
    print(i, " ".join(f"{ev[k][i]:9.0f}" for k in ["issue", "a_ready", "dec_done", "b_ready", "mma"]))
if t.shape[0] > 8:
    nm = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    roles = (["prod"] * 4 + ["dec"] * 4 + ["mma"] * nm + ["epi"] * 4)
    print("per-warp mbarrier wait share (CTA 0):")
    for w in range(len(roles)):
        wt, tot = raw.reshape(-1, N)[8][2 * w], raw.reshape(-1, N)[8][2 * w + 1]
        if tot > 0:
            print(f"  warp {w:2d} {roles[w]:4s}: waiting {100.0 * wt / tot:5.1f}% of {tot} cycles")
