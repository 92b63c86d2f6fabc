"""Summarise ncu --set full reports into a markdown table + the per-kernel DRAM traffic JSON bench.py reads.

usage: python tools/ncu_summary.py OUT_MD WORKLOAD_TAG REP [REP ...] [--traffic]
(--traffic also records each kernel's DRAM bytes per launch in profiles/ncu_traffic.json under
 [WORKLOAD_TAG][kernel name], the key bench.py looks up: tag = "<config>_N<N>_tm<TM>", e.g. c3_N256_tm16)
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
           "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def read(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                v = r[i].replace(",", "")
                try:
                    d[m] = float(v) * SCALE.get(units[i], 1)
                except ValueError:
                    d[m] = v
        res.append(d)
    return res


def main():
    args = [a for a in sys.argv[1:] if a != "--traffic"]
    write_traffic = "--traffic" in sys.argv
    out_md, tag, reps = args[0], args[1], args[2:]
    rows = [d for rep in reps for d in read(rep)]
    lines = [f"\n**{tag}**\n", "| kernel | time us | DRAM read MB | DRAM write MB | DRAM % | L2 % | L2 hit % | L1 % | SM % | tensor % | warps % | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic_path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                                "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    for d in rows:
        g = lambda k: d.get(k, float("nan"))
        lines.append(f"| {d['kernel']} | {g('gpu__time_duration.sum')*1e6:.1f} | {g('dram__bytes_read.sum')/1e6:.1f} | "
                     f"{g('dram__bytes_write.sum')/1e6:.1f} | {g('dram__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | {g('lts__t_sector_hit_rate.pct'):.1f} | "
                     f"{g('l1tex__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | {g('sm__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{g('sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed'):.2f} | "
                     f"{g('sm__warps_active.avg.pct_of_peak_sustained_active'):.1f} | {g('launch__registers_per_thread'):.0f} | "
                     f"{g('launch__grid_size'):.0f} x {g('launch__block_size'):.0f} |")
        name = d["kernel"].replace("void ", "").split("::")[-1].split("<")[0].strip()
        traffic.setdefault(tag, {})[name] = {
            "dram_bytes_per_launch": int(g("dram__bytes_read.sum") + g("dram__bytes_write.sum")),
            "ncu_time_us": round(g("gpu__time_duration.sum") * 1e6, 2)}
    open(out_md, "a").write("\n".join(lines) + "\n")
    if write_traffic:
        json.dump(traffic, open(traffic_path, "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
