"""Turn gpurun_out/prof (ncu reports + launch lists) into committed text/JSON
summaries under profiles/ (CPU side; needs the ncu CLI only)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")
TAG = sys.argv[1] if len(sys.argv) > 1 else "r01"
os.makedirs(DST, exist_ok=True)


def launches(name):
    rows = list(csv.reader(open(os.path.join(SRC, f"launches_{name}.csv"))))
    h = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hd = rows[h]
    ki, vi, ui = hd.index("Kernel Name"), hd.index("Metric Value"), hd.index("Metric Unit")
    out = []
    for r in rows[h + 1:]:
        v = float(r[vi].replace(",", ""))
        us = v / 1000 if r[ui] == "ns" else v * 1000 if r[ui] == "ms" else v
        out.append((r[ki], us))
    return out


summary = {}
for cfg in ("c2", "c3", "c4"):
    if not os.path.exists(os.path.join(SRC, f"launches_{cfg}.csv")):
        continue
    ls = launches(cfg)
    with open(os.path.join(DST, f"{TAG}_launches_{cfg}.txt"), "w") as fh:
        fh.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none, bench.py --config {cfg} "
                 "--steps 2 --warmup 3 (cold-cache, serialised launches)\n")
        ours = [(k, t) for k, t in ls if any(s in k for s in ("attn_", "quantize", "bwd_pre", "dq_convert"))]
        per_step = {"c2": 4, "c3": 4, "c4": 6}[cfg]
        # the full-size timed step: the launches ending at the longest attention launch
        # (later, shorter launches are the host-pipelined e2e chunks)
        # (a full step starts with the quantizers; the roofline loop re-runs the attention kernel alone)
        cand = [i for i in range(per_step - 1, len(ours)) if "attn_" in ours[i][0]
                and "quantize" in ours[i - per_step + 1][0]
                and sum("attn_" in ours[j][0] for j in range(i - per_step + 1, i + 1)) == {"c2": 1, "c3": 1, "c4": 2}[cfg]]
        end = max(cand, key=lambda i: ours[i][1])
        step = ours[max(0, end + 1 - per_step):end + 1]
        tot = sum(t for _, t in step) or 1
        for k, t in ls:
            fh.write(f"{t:12.1f} us  {k[:110]}\n")
        fh.write("\n# share of one full-size step's own kernels (the e2e chunk launches follow it above):\n")
        for k, t in step:
            fh.write(f"{100 * t / tot:6.1f}%  {t:10.1f} us  {k[:90]}\n")

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__issue_active.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.per_cycle_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum"]
if os.path.exists(os.path.join(SRC, "launches_sage3_c2.csv")):
    with open(os.path.join(DST, f"{TAG}_launches_sage3_c2.txt"), "w") as fh:
        fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none, scripts/prof_sage3.py (C2 shape: "
                 "K4 training, K5, then sage3 with no toggles / smoothing / two-level P / all)\n")
        for k, t in launches("sage3_c2"):
            if "at::" not in k:
                fh.write(f"{t:12.1f} us  {k[:110]}\n")

for rep in ("attn_fwd_c2", "attn_fwd_c3", "attn_fwd_train_c4", "attn_bwd_c4", "attn_bwd_plain_c4", "quantize_c2",
            "fp4mm_8k", "attn_fwd_sage3_c2", "attn_fwd_plain_c2", "attn_fwd_mx_c2"):
    path = os.path.join(SRC, rep + ".ncu-rep")
    if not os.path.exists(path):
        continue
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(raw)))
    h, units = r[0], r[1]
    txt = [f"# ncu --set full --clock-control none --import-source on ({rep})"]
    for v in r[2:]:
        d = dict(zip(h, v))
        name = d.get("Kernel Name", "")
        txt.append(f"kernel: {name}")
        for k in KEYS:
            if k in d:
                txt.append(f"  {k:70s} {d[k]} {units[h.index(k)]}")
        st = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): float(x)
              for k, x in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
              and k.endswith("per_issue_active.ratio")}
        txt.append("  stalls/issue: " + ", ".join(f"{a}={b:.2f}" for a, b in sorted(st.items(), key=lambda t: -t[1])
                                                  if b > 0.05))

        def num(k):
            return float(d[k].replace(",", ""))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rb = num("dram__bytes_read.sum") * scale[units[h.index("dram__bytes_read.sum")]]
        wb = num("dram__bytes_write.sum") * scale[units[h.index("dram__bytes_write.sum")]]
        summary.setdefault(rep, []).append({"kernel": name, "dram_bytes_per_launch": rb + wb,
                                            "duration": d["gpu__time_duration.sum"],
                                            "duration_unit": units[h.index("gpu__time_duration.sum")]})
    with open(os.path.join(DST, f"{TAG}_ncu_{rep}.txt"), "w") as fh:
        fh.write("\n".join(txt) + "\n")

# bench.py reads profiles/ncu_summary.json for roofline.traffic (config -> dominant kernel);
# a partial capture updates the existing entries
jpath = os.path.join(DST, "ncu_summary.json")
prev = json.load(open(jpath)) if os.path.exists(jpath) else {}
bench_map = {c: prev[c] for c in ("c2", "c3", "c4", "train_fwd_c4") if c in prev}
for cfg, rep in (("c2", "attn_fwd_c2"), ("c3", "attn_fwd_c3"), ("c4", "attn_bwd_c4"),
                 ("train_fwd_c4", "attn_fwd_train_c4")):
    if rep in summary:
        bench_map[cfg] = summary[rep][0]
allmap = dict(prev.get("all", {}))
allmap.update(summary)
with open(jpath, "w") as fh:
    json.dump({"round": TAG, **bench_map, "all": allmap}, fh, indent=1)
print("wrote", sorted(os.listdir(DST)))
