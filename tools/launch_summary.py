"""Mean duration per kernel of an ncu --metrics gpu__time_duration.sum CSV."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, agg = None, collections.OrderedDict()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        agg.setdefault(d["Kernel Name"][:100], []).append(float(d["Metric Value"].replace(",", "")))
for k, v in agg.items():
    print(f"{len(v):4d} x {sum(v) / len(v) / 1000:8.1f} us  {k}")
