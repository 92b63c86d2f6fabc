"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: per kernel count / mean / share."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    i = next(k for k, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[i], rows[i + 1:]
    ki, mi, ni, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("Metric Unit")
    t = defaultdict(list)
    for r in data:
        if len(r) > mi and r[ni] == "gpu__time_duration.sum":
            v = float(r[mi].replace(",", ""))
            v = v / 1e3 if r[ui] == "ns" else (v * 1e3 if r[ui] == "ms" else v)
            t[r[ki].split("(")[0][:48]].append(v)
    tot = sum(sum(v) for v in t.values())
    print(f"{'kernel':48s} {'n':>4s} {'mean_us':>10s} {'share':>7s}")
    for k, v in sorted(t.items(), key=lambda x: -sum(x[1])):
        print(f"{k:48s} {len(v):4d} {sum(v)/len(v):10.1f} {sum(v)/tot:7.3f}")


if __name__ == "__main__":
    main(sys.argv[1])
