"""Windowed stall map of an ncu report's SASS (CPU side):
    python scripts/stall_map.py rep.ncu-rep [window]
For every window of SASS instructions: share of all stall samples, the top
stall reasons, instructions executed and a few representative opcodes."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
win = int(sys.argv[2]) if len(sys.argv) > 2 else 40
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(x for x in rows if "Source" in x and "Instructions Executed" in x)
body = [r for r in rows[rows.index(hdr) + 1:] if len(r) == len(hdr)]
si, ti, ei = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[ti] or 0) for r in body) or 1
print(f"total samples {tot}, {len(body)} instructions")
agg = collections.Counter()
for r in body:
    for h in reasons:
        agg[h] += int(r[hdr.index(h)] or 0)
print("overall:", ", ".join(f"{k[6:]} {100*v/tot:.1f}%" for k, v in agg.most_common(8)))
for w0 in range(0, len(body), win):
    ch = body[w0:w0 + win]
    s = sum(int(r[ti] or 0) for r in ch)
    if s < 0.01 * tot:
        continue
    c = collections.Counter()
    for r in ch:
        for h in reasons:
            c[h] += int(r[hdr.index(h)] or 0)
    ex = max(int(r[ei] or 0) for r in ch)
    ops = collections.Counter(r[si].split()[0] if not r[si].strip().startswith("@") else r[si].split()[1] for r in ch)
    print(f"[{w0:5d}-{w0 + len(ch) - 1:5d}] {100 * s / tot:5.1f}%  ex<={ex:>8d}  "
          + ", ".join(f"{k[6:]} {100 * v / s:.0f}%" for k, v in c.most_common(3))
          + "  | " + " ".join(f"{o.split('.')[0]}x{n}" for o, n in ops.most_common(5)))
