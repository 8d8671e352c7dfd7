"""Per-source-line warp-stall samples of one kernel from `ncu -i X.ncu-rep --page source --csv
--print-source cuda,sass` (stdin or a file): the top lines with their dominant stall reasons."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr, fname, lines = None, None, []
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr[4:], r[4:]))
        n = int(d["# Samples"] or 0)
        if n:
            st = sorted(((int(d[k] or 0), k) for k in hdr if k.startswith("stall_") and "Not Issued" not in k), reverse=True)[:3]
            lines.append((n, fname, r[0], r[1].strip()[:90], ", ".join(f"{k[6:]} {v}" for v, k in st if v),
                          int(d["Instructions Executed"] or 0)))
tot = sum(l[0] for l in lines)
print(f"total samples {tot}")
for n, f, ln, src, st, ins in sorted(lines, reverse=True)[:top]:
    print(f"{100.0 * n / tot:5.1f}%  {f}:{ln:>4s}  inst {ins:>10d}  [{st}]  {src}")
