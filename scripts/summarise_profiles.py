"""Turn gpurun_out/ ncu reports of one tag into the tracked summaries under profiles/.

    python scripts/summarise_profiles.py r1d r1      # <gpurun tag> <profiles prefix>
"""
import collections
import csv
import json
import os
import shutil
import subprocess
import sys

tag, out = sys.argv[1], sys.argv[2]
G, P = "gpurun_out", "profiles"
os.makedirs(P, exist_ok=True)

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
]


def raw(report):
    txt = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    return hdr, units, rows[2:]


def summarise(report, dest):
    hdr, units, rows = raw(report)
    idx = {h: i for i, h in enumerate(hdr)}
    lines = [f"# {os.path.basename(report)}: ncu --set full --clock-control none (per launch, cold cache, serialised)"]
    for r in rows:
        lines.append(f"\n## {r[idx['Kernel Name']]}  (launch id {r[idx['ID']]})")
        for m in METRICS:
            if m in idx:
                lines.append(f"{m:90s} {r[idx[m]]:>18s} {units[idx[m]]}")
    open(dest, "w").write("\n".join(lines) + "\n")
    return hdr, units, rows, idx


# launch list -> shares
rows = list(csv.reader(open(f"{G}/launches_{tag}.csv")))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
ki, vi = rows[h].index("Kernel Name"), rows[h].index("Metric Value")
agg = collections.OrderedDict()
for r in rows[h + 1:]:
    if len(r) > vi:
        a = agg.setdefault(r[ki], [0, 0.0])
        a[0] += 1
        a[1] += float(r[vi].replace(",", ""))
tot = sum(v[1] for v in agg.values())
with open(f"{P}/{out}_launches.csv", "w") as fh:
    fh.write("# ncu --metrics gpu__time_duration.sum --clock-control none: python bench.py --steps 5 --warmup 3 --skip-cpu\n")
    fh.write("kernel,launches,total_us,share_pct\n")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        fh.write(f"\"{k}\",{v[0]},{v[1] / 1e3:.1f},{100 * v[1] / tot:.2f}\n")

hdr, units, srows, idx = summarise(f"{G}/prof_stencil_{tag}.ncu-rep", f"{P}/{out}_stencil_ncu.txt")
r = srows[-1]
to_b = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rd = float(r[idx["dram__bytes_read.sum"]]) * to_b[units[idx["dram__bytes_read.sum"]]]
wr = float(r[idx["dram__bytes_write.sum"]]) * to_b[units[idx["dram__bytes_write.sum"]]]
bench = json.load(open(f"{G}/bench_{tag}.json"))
json.dump({"stencils": bench["config"]["stencils_per_gpu"], "dram_bytes_per_step": rd + wr, "dram_read": rd,
           "dram_write": wr, "kernel_us_under_ncu": float(r[idx["gpu__time_duration.sum"]]),
           "source": f"{out}_stencil_ncu.txt (one fused launch = one step)"},
          open(f"{P}/stencil_traffic.json", "w"), indent=1)
summarise(f"{G}/prof_newton_{tag}.ncu-rep", f"{P}/{out}_newton_ncu.txt")
shutil.copy(f"{G}/bench_{tag}.json", f"{P}/{out}_bench.json")
if os.path.exists(f"{G}/bench_{tag}_ref.json"):
    shutil.copy(f"{G}/bench_{tag}_ref.json", f"{P}/{out}_bench_reference_arm.json")
print(open(f"{P}/{out}_launches.csv").read()[:1800])
print(open(f"{P}/stencil_traffic.json").read())
