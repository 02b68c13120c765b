"""Aggregate an ncu report's warp-stall samples per CUDA source line.

usage: python tools/ncu_lines.py REPORT.ncu-rep [top_n] [column]
column: a source-page metric column name (default: the warp-stall samples,
column 4), e.g. "Instructions Executed".
Prints the hottest source lines (file:line, samples, share, source text).
Needs the report captured with -lineinfo builds and --import-source on.
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    col = sys.argv[3] if len(sys.argv) > 3 else None
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, total, path, hdr = {}, 0, "?", None
    cur = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            path = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 5:
            continue
        if r[0]:
            cur = (path, r[0], r[1])
            ci = hdr.index(col) if (col and col in hdr) else 4
            try:
                v = int(float(r[ci] or 0))
            except ValueError:
                v = 0
            agg[cur] = agg.get(cur, 0) + v
            total += v
    items = sorted(agg.items(), key=lambda kv: -kv[1])[:top]
    print(f"total {col or 'samples'} {total}")
    for (p, ln, src), v in items:
        print(f"{v:7d} {100.0 * v / max(total, 1):5.1f}%  {p}:{ln}  {src.strip()[:110]}")


if __name__ == "__main__":
    main()
