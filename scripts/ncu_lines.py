"""Aggregate an ncu `--page source --print-source cuda,sass --csv` dump per CUDA source line."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
rows = list(csv.reader(open(path)))
cur_file, out = None, []
hdr = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0] != "":
        d = dict(zip(hdr[2:], r[2:]))
        try:
            out.append((int(d["Warp Stall Sampling (All Samples)"]), int(d["Instructions Executed"]), cur_file, r[0],
                        r[1].strip()[:90]))
        except (KeyError, ValueError):
            pass
tot_s = sum(o[0] for o in out) or 1
tot_i = sum(o[1] for o in out) or 1
print(f"total samples {tot_s}, warp instructions {tot_i}")
for s, i, f, ln, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot_s:5.1f}% smp {100 * i / tot_i:5.1f}% inst  {f}:{ln}  {src}")
