"""Per-SASS-instruction view of an ncu report: python tools/ncu_sass.py REP [column] [top]
Aggregates the column (default 'Warp Stall Sampling (All Samples)') by opcode and lists
the top instructions with their CUDA source line."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "Warp Stall Sampling (All Samples)"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
items = []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    d = dict(zip(hdr, r))
    try:
        v = float(d.get(col, "0") or 0)
    except ValueError:
        v = 0.0
    items.append((v, d.get("Address"), d.get("Source", "")))
tot = sum(v for v, _, _ in items) or 1.0
byop = collections.Counter()
for v, _, src in items:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    byop[op.split(".")[0]] += v
print(f"total {col}: {tot:.0f}")
for op, v in byop.most_common(20):
    print(f"  {v / tot * 100:5.1f}%  {op}")
print("top instructions:")
for v, a, src in sorted(items, key=lambda t: -t[0])[:top]:
    print(f"  {v / tot * 100:5.1f}%  {a}  {src[:100]}")
