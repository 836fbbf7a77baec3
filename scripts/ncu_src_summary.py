"""Summarise an `ncu --page source --csv --print-source cuda,sass` export:
the source lines with the most warp-stall samples and their main stall
reasons, plus the kernel-wide stall mix.

    python scripts/ncu_src_summary.py gpurun_out/src_single_nw1.csv [top]
"""
import csv
import sys
from collections import defaultdict


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    cur_file, header = None, None
    lines = defaultdict(lambda: [0, defaultdict(int), ""])
    total = defaultdict(int)
    with open(path, newline="") as f:
        for row in csv.reader(f):
            if not row:
                continue
            if row[0] == "File Path":
                cur_file = row[1].split("/")[-1]
                continue
            if row[0] == "Function Name":
                continue
            if row[0] == "Line No":
                header = row
                continue
            if header is None or not row[0] or row[0] == "":
                continue
            try:
                n = int(row[4])
            except ValueError:
                continue
            key = (cur_file, int(row[0]))
            e = lines[key]
            e[0] += n
            e[2] = row[1][:90]
            for i, h in enumerate(header):
                if h.startswith("stall_") and "Not Issued" not in h:
                    try:
                        v = int(row[i])
                    except ValueError:
                        continue
                    e[1][h] += v
                    total[h] += v
    allsum = sum(e[0] for e in lines.values()) or 1
    print(f"total samples {allsum}")
    ts = sum(total.values()) or 1
    print("stall mix: " + ", ".join(f"{k[6:]} {100 * v / ts:.1f}%" for k, v in
                                   sorted(total.items(), key=lambda kv: -kv[1])[:8]))
    for (fn, ln), (n, st, src) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        s = sum(st.values()) or 1
        mix = ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:3])
        print(f"{100 * n / allsum:5.1f}% {fn}:{ln:<5d} {src:<90s} [{mix}]")


if __name__ == "__main__":
    main()
