"""Warp-stall breakdown (per issued instruction) of an ncu report: python tools/ncu_stalls.py REP"""
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, v = rows[0], rows[2]
d = dict(zip(h, v))
st = []
for k in h:
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
        try:
            st.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(d[k])))
        except ValueError:
            pass
tot = sum(x for _, x in st)
print(f"total stall cycles per issued instruction: {tot:.2f}")
for k, x in sorted(st, key=lambda t: -t[1]):
    if x > 0.02:
        print(f"  {x:6.2f}  {k}")
