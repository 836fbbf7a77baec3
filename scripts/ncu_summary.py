"""Markdown table of the key metrics of an ncu `--page raw --csv` export (one kernel)."""
import csv
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]

rows = list(csv.reader(open(sys.argv[1])))
h, units, v = rows[0], rows[1], rows[2]
d = {k: (x, u) for k, u, x in zip(h, units, v)}
print(f"Kernel: `{d.get('Kernel Name', ('?', ''))[0]}`\n")
print("| metric | value | unit |\n|---|---|---|")
for k in KEYS:
    if k in d:
        print(f"| {k} | {d[k][0]} | {d[k][1]} |")
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(x) for k, (x, _) in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and x.isdigit()}
tot = sum(st.values()) or 1
print("\nWarp-stall samples (top): " + ", ".join(f"{k} {100 * x / tot:.1f}%" for k, x in
                                                   sorted(st.items(), key=lambda kv: -kv[1])[:6]))
