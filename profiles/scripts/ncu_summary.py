"""Summarise an `ncu --csv --metrics ...` log: one line per kernel launch."""
import csv
import sys

rows = [l for l in open(sys.argv[1]) if l.startswith('"')]
r = list(csv.reader(rows))
h = r[0]
out = {}
for row in r[1:]:
    d = dict(zip(h, row))
    key = (d["ID"], d["Kernel Name"][:48], d["Grid Size"])
    out.setdefault(key, {})[d["Metric Name"]] = d["Metric Value"]
for (i, k, g), m in out.items():
    t = float(m.get("gpu__time_duration.sum", "nan")) / 1e3
    rd = float(m.get("dram__bytes_read.sum", "nan")) / 1e6
    wr = float(m.get("dram__bytes_write.sum", "nan")) / 1e6
    f64 = m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_elapsed", "")
    print(f"{i:>3} {k:48s} {g:>14s} {t:9.1f} us  rd {rd:9.2f} MB  wr {wr:9.2f} MB  fp64 {f64}%")
