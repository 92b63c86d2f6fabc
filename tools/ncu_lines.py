"""Warp-stall samples per CUDA source line of one kernel, from `ncu -i REP --page source --print-source cuda,sass`.

usage: python tools/ncu_lines.py REP KERNEL_REGEX [N]
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    st = next(i for i, l in enumerate(lines) if l.startswith('"Line No"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[st:]))))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    agg, txt = defaultdict(float), {}
    for r in rows[1:]:  # source-line rows carry the line's aggregate; the SASS rows under them are skipped
        if len(r) <= si or not r[0].strip().isdigit():
            continue
        ln = int(r[0])
        txt[ln] = r[1].strip()[:110]
        try:
            agg[ln] += float(r[si] or 0)
        except ValueError:
            pass
    tot = sum(agg.values()) or 1
    for ln, v in sorted(agg.items(), key=lambda x: -x[1])[:n]:
        print(f"{100 * v / tot:6.2f}%  L{ln}  {txt.get(ln, '')}")


if __name__ == "__main__":
    main()
