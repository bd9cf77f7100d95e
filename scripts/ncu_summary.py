"""Summarise an ncu report: key throughput metrics, stall reasons, opcode mix (CPU side)."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, units = r[0], r[1]
for v in r[2:]:
    d = dict(zip(h, v))
    print("kernel:", d.get("Kernel Name", "")[:90])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
            "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
            "launch__registers_per_thread", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
    for k in keys:
        if k in d:
            print(f"  {k:70s} {d[k]} {units[h.index(k)]}")
    st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(x)
          for k, x in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
    print("  stalls/issue:", ", ".join(f"{k}={v:.2f}" for k, v in sorted(st.items(), key=lambda t: -t[1]) if v > 0.05))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = next(x for x in rows if "Source" in x and "Instructions Executed" in x)
si, ei, sti = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
cnt, stall = collections.Counter(), collections.Counter()
for row in rows[rows.index(hdr) + 1:]:
    if len(row) <= ei or not row[si].strip():
        continue
    toks = row[si].strip().split()
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    op = op.split(".")[0]
    try:
        cnt[op] += int(row[ei])
        stall[op] += int(row[sti])
    except ValueError:
        pass
tot = sum(cnt.values())
tst = sum(stall.values()) or 1
print("  opcode mix (share of executed warp instructions, share of stall samples):")
for op, c in cnt.most_common(16):
    print(f"    {op:10s} {100 * c / tot:5.1f}%  stalls {100 * stall[op] / tst:5.1f}%")
