"""Summarise an ncu ``--page source --csv --print-source sass`` dump.

    python scripts/sass_hist.py gpurun_out/prof/fwd_c2_sass.csv [--listing lo hi] [--hot]

Prints dynamic warp-instruction counts per opcode and the stall-sample
histogram, plus (``--listing``) the annotated SASS between two row indices.
"""
import csv
import sys
from collections import Counter, defaultdict


def load(path):
    with open(path) as fh:
        rows = list(csv.reader(fh))
    hdr_i = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
    hdr = rows[hdr_i]
    out = []
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        out.append(dict(zip(hdr, r)))
    return hdr, out


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


def main():
    path = sys.argv[1]
    hdr, rows = load(path)
    ops = Counter()
    samples = Counter()
    stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    stalls = defaultdict(float)
    total = 0
    for r in rows:
        src = r["Source"].strip()
        op = src.split()[0] if src else "?"
        if op.startswith("@"):
            op = src.split()[1]
        base = op.split(".")[0]
        n = num(r["Instructions Executed"])
        ops[base] += n
        total += n
        samples[base] += num(r["Warp Stall Sampling (All Samples)"])
        for c in stall_cols:
            stalls[c] += num(r[c])
    print(f"total warp instructions executed: {total:.4g}")
    for op, n in ops.most_common(40):
        print(f"  {op:12s} {n:14.4g}  {100 * n / total:5.1f}%   samples {samples[op]:8.0f}")
    tot_s = sum(stalls.values())
    print("stall samples:")
    for c, v in sorted(stalls.items(), key=lambda kv: -kv[1])[:14]:
        print(f"  {c:28s} {v:10.0f} {100 * v / tot_s:5.1f}%")
    if "--listing" in sys.argv:
        i = sys.argv.index("--listing")
        lo, hi = int(sys.argv[i + 1]), int(sys.argv[i + 2])
        for k, r in enumerate(rows[lo:hi], lo):
            print(f"{k:5d} {num(r['Instructions Executed']):12.0f} {num(r['Warp Stall Sampling (All Samples)']):7.0f}  "
                  f"{r['Source'].strip()}")
    if "--hot" in sys.argv:
        best = sorted(range(len(rows)), key=lambda k: -num(rows[k]["Warp Stall Sampling (All Samples)"]))[:40]
        for k in sorted(best):
            r = rows[k]
            print(f"{k:5d} {num(r['Instructions Executed']):12.0f} {num(r['Warp Stall Sampling (All Samples)']):7.0f}  "
                  f"{r['Source'].strip()}")


if __name__ == "__main__":
    main()
