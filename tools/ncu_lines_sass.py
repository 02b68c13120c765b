"""Per-CUDA-line totals of a SASS-level column (default "Instructions Executed"),
attributing each SASS row to the CUDA line printed above it:
python tools/ncu_lines_sass.py REP [column] [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
col = sys.argv[2] if len(sys.argv) > 2 else "Instructions Executed"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
hdr, cur, path, agg, tot = None, None, "?", {}, 0.0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Name":
        path = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) != len(hdr):
        continue
    if r[0]:
        cur = (path, r[0], r[1])
        continue
    if r[2] in ("", "..."):
        continue
    try:
        v = float(r[hdr.index(col, 4)] or 0)
    except ValueError:
        continue
    agg[cur] = agg.get(cur, 0.0) + v
    tot += v
print(f"total {col}: {tot:.0f}")
for (p, ln, src), v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:10.0f} {100 * v / max(tot, 1):5.1f}%  {p}:{ln}  {src.strip()[:100]}")
