"""profiles/sweep_traffic.json from an ncu --set full raw CSV of the headline
sweep kernel: DRAM bytes per launch and the SASS hash of the captured build
(bench.py compares it with the build it times)."""
import csv
import json
import sys

sys.path.insert(0, ".")
from bench import sweep_sass_sha256  # noqa: E402

rows = list(csv.reader(open(sys.argv[1])))
d = dict(zip(rows[0], rows[2]))
units = dict(zip(rows[0], rows[1]))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(d["dram__bytes_read.sum"]) * scale[units["dram__bytes_read.sum"]]
wr = float(d["dram__bytes_write.sum"]) * scale[units["dram__bytes_write.sum"]]
out = {"dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
       "gpu_time_us": float(d["gpu__time_duration.sum"]) * (1e3 if units["gpu__time_duration.sum"] == "ms" else 1),
       "kernel": d.get("Kernel Name"), "sass_sha256": sweep_sass_sha256(),
       "source": sys.argv[2] if len(sys.argv) > 2 else "ncu --set full, 1 launch, cold cache, clocks unlocked"}
json.dump(out, open("profiles/sweep_traffic.json", "w"), indent=1)
print(out)
