"""Executed warp instructions per CUDA source line of an ncu report.

usage: python tools/ncu_inst.py REPORT.ncu-rep [top_n]
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    path, agg = "?", {}
    for r in csv.reader(io.StringIO(out)):
        if not r or r[0] in ("Line No", "Function Name"):
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] and len(r) > 7:
            try:
                ie = int(float(r[7] or 0))
            except ValueError:
                ie = 0
            k = (path, r[0], r[1].strip()[:100])
            agg[k] = agg.get(k, 0) + ie
    tot = sum(agg.values())
    print(f"total warp instructions {tot}")
    for (p, ln, src), ie in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
        print(f"{ie:10d} {100.0 * ie / max(tot, 1):5.1f}%  {p}:{ln}  {src}")


if __name__ == "__main__":
    main()
