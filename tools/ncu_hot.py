"""Top SASS lines by warp-stall samples from an .ncu-rep (source page)."""
import csv
import io
import subprocess
import sys

rep, n = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, iss, iex = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), \
    h.index("Instructions Executed")
data = []
for r in rows[2:]:
    try:
        data.append((int(r[iss] or 0), r[ia], r[isrc], r[iex]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for s, a, src, ex in sorted(data, reverse=True)[:n]:
    print(f"{100 * s / tot:5.1f}%  {a}  {src[:90]:90s} exec={ex}")
