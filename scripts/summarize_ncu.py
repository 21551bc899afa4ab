"""Summarise ncu outputs from gpurun_out/ into profiles/<round>/ (committed evidence)."""
import collections
import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
RUN = sys.argv[1] if len(sys.argv) > 1 else "round1"
SRC = os.path.join(ROOT, "gpurun_out")
# optional second argument: output directory (on the GPU box: a gpurun_out/ subdirectory, so the
# summaries travel back without the large .ncu-rep files)
DST = sys.argv[2] if len(sys.argv) > 2 else os.path.join(ROOT, "profiles", RUN)
os.makedirs(DST, exist_ok=True)

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x",
        "sm__cycles_elapsed.avg.per_second", "smsp__inst_executed.sum"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    if len(rows) < 3:
        return []
    h, u = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")]}
        for k in KEYS:
            if k in h:
                d[k] = f"{r[h.index(k)]} {u[h.index(k)]}".strip()
        res.append(d)
    return res


# merge: captures present in gpurun_out/ replace their entries, the others are kept
out_json = os.path.join(DST, "ncu_full_summary.json")
summary = json.load(open(out_json)) if os.path.exists(out_json) else {}
for rep in sorted(glob.glob(os.path.join(SRC, "full_*.ncu-rep"))):
    summary[os.path.basename(rep)] = raw(rep)
json.dump(summary, open(os.path.join(DST, "ncu_full_summary.json"), "w"), indent=1)

lst = os.path.join(SRC, "launches_r1.csv")
if os.path.exists(lst):
    rows = list(csv.reader(open(lst)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ik, iv, iu = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    with open(os.path.join(DST, "launches.csv"), "w") as f:
        f.write("id,kernel,duration_us\n")
        for r in rows[hi + 1:]:
            if len(r) <= iv:
                continue
            v = float(r[iv].replace(",", ""))
            v = v / 1000 if r[iu] == "ns" else v * 1000 if r[iu] == "ms" else v
            name = r[ik].split("(")[0].replace("void ", "")
            f.write(f"{r[0]},\"{name}\",{v:.3f}\n")
            agg[name][0] += 1
            agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    with open(os.path.join(DST, "launches_by_kernel.txt"), "w") as f:
        f.write("ncu --metrics gpu__time_duration.sum --clock-control none python bench.py --steps 2 --warmup 3 "
                "--no-cpu-baseline --no-graphs\n")
        f.write("(cold-cache, serialised launches: compare shares, not absolute times)\n\n")
        for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
            f.write(f"{k[:80]:80s} launches={v[0]:5d} total_us={v[1]:11.1f} share={v[1] / tot:.3f}\n")
print("wrote", DST)
