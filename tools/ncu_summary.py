"""Per-launch kernel times from an ncu --csv launch list (gpu__time_duration):
python tools/ncu_summary.py launches.csv [min_ns] [from_kernel_substring]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 50000
start_pat = sys.argv[3] if len(sys.argv) > 3 else None
hdr, out = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        out.append((d["Kernel Name"][:70], float(d["Metric Value"].replace(",", ""))))
start = 0
if start_pat:
    idx = [i for i, (nm, _) in enumerate(out) if start_pat in nm]
    start = idx[-1] if idx else 0
for nm, v in out[start:]:
    if v > mn:
        print(f"{v / 1e6:10.3f} ms  {nm}")
