"""Summarize an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections
import csv
import sys


def summarize(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in data:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].split("::")[-1]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"{'kernel':32s} {'launches':>8s} {'total_us':>10s} {'share':>6s} {'avg_us':>8s}"]
    for k, v in sorted(tot.items(), key=lambda t: -t[1]):
        lines.append(f"{k:32s} {cnt[k]:8d} {v / 1e3:10.1f} {v / T * 100:5.1f}% {v / cnt[k] / 1e3:8.2f}")
    lines.append(f"total {T / 1e6:.3f} ms over {sum(cnt.values())} launches (cold-cache, serialised)")
    return "\n".join(lines)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
