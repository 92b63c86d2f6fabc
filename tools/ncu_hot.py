"""Top source lines of a kernel by warp-stall samples, from `ncu -i rep --page source --csv`.

usage: python tools/ncu_hot.py REP KERNEL_REGEX [N] [--sass]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 and sys.argv[3].isdigit() else 25
    mode = "sass"
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern,
                          "--print-source", mode], capture_output=True, text=True).stdout
    lines = out.splitlines()
    # skip the kernel-name line(s)
    start = next(i for i, l in enumerate(lines) if l.startswith('"Address"') or l.startswith('"Line"') or
                 l.startswith('"#"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
    h = rows[0]
    si = h.index("Warp Stall Sampling (All Samples)")
    src = h.index("Source")
    ie = h.index("Instructions Executed") if "Instructions Executed" in h else None
    data = []
    for r in rows[1:]:
        try:
            data.append((float(r[si] or 0), r[src].strip()[:110], r[ie] if ie is not None else "", r[0]))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    for s, txt, ex, addr in sorted(data, reverse=True)[:n]:
        print(f"{100*s/tot:6.2f}%  {ex:>12s}  {addr:>6s}  {txt}")


if __name__ == "__main__":
    main()
