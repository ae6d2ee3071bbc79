"""Summarise an ncu --csv launch list (gpu__time_duration / dram bytes per launch)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID") + 1
hdr = rows[start - 1]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
cur = {}
for r in rows[start:]:
    if len(r) < len(hdr):
        continue
    cur.setdefault((int(r[0]), r[ki].split("(")[0][:48]), {})[r[mi]] = float(r[vi].replace(",", ""))
for (i, k), m in sorted(cur.items()):
    t = m.get("gpu__time_duration.sum", 0) / 1e3
    rd, wr = m.get("dram__bytes_read.sum", 0) / 1e6, m.get("dram__bytes_write.sum", 0) / 1e6
    print(f"{i:3d} {k:48s} {t:9.1f} us  rd {rd:8.1f} MB  wr {wr:8.1f} MB  {(rd + wr) / max(t, 1e-9):6.2f} TB/s")
