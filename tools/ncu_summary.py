"""Summarise an ncu --set full report: per kernel, time, DRAM traffic, issue
utilisation, occupancy and the top stall reasons.  Usage:
    python tools/ncu_summary.py REPORT.ncu-rep [algorithmic_bytes_per_launch]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "dram throughput %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__cluster_dim_x", "cluster x"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
]


def main():
    rep = sys.argv[1]
    alg = float(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {k: i for i, k in enumerate(hdr)}
    for r in data:
        name = r[col["Kernel Name"]]
        print(f"== {name[:110]}")
        vals = {}
        for k, label in KEYS:
            if k in col:
                vals[k] = r[col[k]]
                print(f"   {label:24s} {r[col[k]]:>16s} {units[col[k]]}")
        try:
            t_us = float(vals["gpu__time_duration.sum"])
            t_unit = units[col["gpu__time_duration.sum"]]
            t_s = t_us * {"usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(t_unit, 1e-6)
            scale = {"Mbyte": 1e6, "Gbyte": 1e9, "Kbyte": 1e3, "byte": 1.0}
            rd = float(vals["dram__bytes_read.sum"]) * scale.get(units[col["dram__bytes_read.sum"]], 1.0)
            wr = float(vals["dram__bytes_write.sum"]) * scale.get(units[col["dram__bytes_write.sum"]], 1.0)
            print(f"   {'dram traffic':24s} {rd + wr:16.4e} B  -> {(rd + wr) / t_s / 1e9:8.1f} GB/s")
            if alg:
                print(f"   {'algorithmic bytes':24s} {alg:16.4e} B  -> {alg / t_s / 1e9:8.1f} GB/s "
                      f"(traffic / algorithmic = {(rd + wr) / alg:.3f})")
        except (KeyError, ValueError):
            pass
        stalls = []
        for k, i in col.items():
            if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        tot = sum(v for v, _ in stalls) or 1.0
        print("   stalls (warps per issue):", ", ".join(f"{n} {v:.2f} ({v / tot:.0%})" for v, n in stalls[:8]))


if __name__ == "__main__":
    main()
