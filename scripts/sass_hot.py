"""Print the SASS of an ncu report with per-instruction stall samples / executions,
marking the hottest regions (CPU side). usage: sass_hot.py rep.ncu-rep [min_samples]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 200
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(x for x in rows if "Source" in x and "Instructions Executed" in x)
ai, si, ei, sti = (hdr.index(k) for k in ("Address", "Source", "Instructions Executed",
                                          "Warp Stall Sampling (All Samples)"))
body = [r for r in rows[rows.index(hdr) + 1:] if len(r) > sti]
tot = sum(int(r[sti] or 0) for r in body) or 1
for i, r in enumerate(body):
    s = int(r[sti] or 0)
    if s >= thr:
        print(f"{i:5d} {100 * s / tot:5.2f}% ex={r[ei]:>9s}  {r[si].strip()[:90]}")
