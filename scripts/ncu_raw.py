"""Print key metrics + stall breakdown from an ncu --page raw --csv dump."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
for k in ["gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
          "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
          "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
          "launch__block_size", "launch__waves_per_multiprocessor", "dram__bytes_read.sum", "dram__bytes_write.sum",
          "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]:
    print(k, d.get(k))
st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): int(x) for k, x in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and x.isdigit()}
tot = sum(st.values()) or 1
print(sorted([(round(100 * x / tot, 1), k) for k, x in st.items()], reverse=True)[:10])
