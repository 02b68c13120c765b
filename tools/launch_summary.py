"""Per-kernel means of an ncu --metrics CSV (gpu__time_duration.sum, and DRAM
bytes read / written when captured): launches, mean us, MB read / written,
achieved GB/s."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = None
agg = collections.OrderedDict()  # kernel -> metric -> [values]
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        m = agg.setdefault(d["Kernel Name"][:100], collections.OrderedDict())
        m.setdefault(d["Metric Name"], []).append(float(d["Metric Value"].replace(",", "")))
for k, m in agg.items():
    t = m.get("gpu__time_duration.sum")
    if not t:
        continue
    us = sum(t) / len(t) / 1000
    line = f"{len(t):4d} x {us:8.1f} us"
    rd, wr = m.get("dram__bytes_read.sum"), m.get("dram__bytes_write.sum")
    if rd and wr:
        mr, mw = sum(rd) / len(rd) / 1e6, sum(wr) / len(wr) / 1e6
        line += f"  {mr:8.1f} MB rd {mw:7.1f} MB wr  {(mr + mw) / us * 1e3:7.1f} GB/s"
    print(f"{line}  {k}")
