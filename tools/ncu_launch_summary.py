"""Summarise an ncu launch-list CSV (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) per kernel name:
launches, total ms, share of kernel time, DRAM GB."""
import collections
import csv
import sys

path, title = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
iK, iM, iU, iV = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
iID = hdr.index("ID")
per = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    v = float(r[iV].replace(",", ""))
    u = r[iU]
    scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6,
             "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}.get(u, 1.0)
    per[r[iID]][r[iM]] = v * scale
    names[r[iID]] = r[iK].split("(")[0][:42]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i, m in per.items():
    a = agg[names[i]]
    a[0] += 1
    a[1] += m.get("gpu__time_duration.sum", 0.0)
    a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
tot = sum(a[1] for a in agg.values())
print(title)
print(f"total launches {len(per)}, total kernel time {tot:.1f} ms")
print(f"{'kernel':42s} {'launches':>8s} {'ms':>10s} {'share':>6s} {'DRAM GB':>9s}")
for k, (c, ms, gb) in sorted(agg.items(), key=lambda t: -t[1][1]):
    print(f"{k:42s} {c:8d} {ms:10.1f} {100 * ms / tot:5.1f}% {gb:9.2f}")
