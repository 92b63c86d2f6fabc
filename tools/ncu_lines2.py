"""Per-source-line warp-stall samples and executed instructions of one kernel in an ncu report (cuda,sass view).

usage: python tools/ncu_lines2.py REP KERNEL [N]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", kern, "--launch-count", "1",
                          "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, cur_file, cur_line, seen = None, None, None, {}
    for r in rows:
        if r and r[0] == "File Path":
            cur_file = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8:
            continue
        if r[0]:
            cur_line = (cur_file, int(r[0]), r[1].strip()[:90])
        if not r[2].startswith("0x") or r[2] in seen:
            continue
        try:
            seen[r[2]] = (cur_line, float(r[4] or 0), float(r[7] or 0))
        except ValueError:
            pass
    agg = {}
    for cl, st, ex in seen.values():
        a = agg.setdefault(cl, [0.0, 0.0])
        a[0] += st
        a[1] += ex
    ts = sum(v[0] for v in agg.values()) or 1
    te = sum(v[1] for v in agg.values()) or 1
    print(f"{kern}: {te / 1e6:.1f}M warp instructions")
    for cl, v in sorted(agg.items(), key=lambda x: -x[1][0])[:n]:
        if cl:
            print(f"{100 * v[0] / ts:5.1f}% stall {100 * v[1] / te:5.1f}% inst  {cl[0]}:{cl[1]}  {cl[2]}")


if __name__ == "__main__":
    main()
