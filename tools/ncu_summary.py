"""Summaries of ncu exports: `python tools/ncu_summary.py raw <raw.csv>...` (key metrics + top stall
reasons of each captured launch) or `python tools/ncu_summary.py launches <launches.csv>` (time per
kernel over the launch list)."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]


def raw(fn):
    rows = list(csv.reader(open(fn)))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        name = v[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        print("==", fn, name[:90])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:62s} {v[i]} {u[i]}")
        st = [(h[i], float(v[i] or 0)) for i in range(len(h))
              if h[i].startswith("smsp__pcsamp_warps_issue_stalled") and not h[i].endswith("not_issued")]
        tot = sum(x for _, x in st) or 1.0
        for a, b in sorted(st, key=lambda x: -x[1])[:8]:
            print(f"    {a.replace('smsp__pcsamp_warps_issue_stalled_', 'stall_'):50s} {100 * b / tot:5.1f} %")


def launches(fn):
    rows = list(csv.reader(open(fn)))
    for i, r in enumerate(rows):
        if "Kernel Name" in r:
            h, start = r, i + 1
            break
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = {}
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        try:
            v = float(r[vi].replace(",", ""))
        except ValueError:
            continue
        k = r[ki].split("(")[0].split("<")[0]
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += v
    tot = sum(v[1] for v in agg.values())
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:12]:
        print(f"{k:45s} {v[0]:5d} {v[1] / 1e6:10.2f} ms {100 * v[1] / tot:5.1f} %")


if __name__ == "__main__":
    {"raw": lambda fs: [raw(f) for f in fs], "launches": lambda fs: [launches(f) for f in fs]}[sys.argv[1]](sys.argv[2:])
