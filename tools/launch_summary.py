"""Per-kernel totals of an ncu launch list (--metrics gpu__time_duration.sum --csv).
  python tools/launch_summary.py <launches.csv> [top]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, d = rows[0], rows[1:]
ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in d:
    if r[iu] in scale:
        name = r[ik].split("(")[0].replace("fgb::<unnamed>::", "")
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", "")) * scale[r[iu]]
tot = sum(v for _, v in agg.values()) or 1.0
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
print(f"{'share':>7} {'seconds':>9} {'launches':>8}  kernel")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{100 * v / tot:6.2f}% {v:9.3f} {c:8d}  {n}")
print(f"total {tot:.3f} s over {sum(c for c, _ in agg.values())} launches")
