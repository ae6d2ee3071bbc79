"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel launch."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0] != "ID"]
d = collections.OrderedDict()
for r in rows:
    d.setdefault((int(r[0]), r[4].split("(")[0][:60]), {})[r[12]] = float(r[14].replace(",", ""))
tot_t = sum(m.get("gpu__time_duration.sum", 0) for m in d.values())
for (i, k), m in d.items():
    t = m.get("gpu__time_duration.sum", 0)
    print(f"{i:>4} {k:60s} {t / 1e3:9.1f} us {100 * t / tot_t:5.1f}%  rd {m.get('dram__bytes_read.sum', 0) / 2**20:8.1f} MiB"
          f"  wr {m.get('dram__bytes_write.sum', 0) / 2**20:8.1f} MiB")
