"""fp64 flops per launch of the compute-bound kernels, counted by ncu on the GPU box:
2 x DFMA + DADD + DMUL thread-level instructions of accd_kernel (the CCD filter of the bench's cloth stack)
and the two elastic kernels (400 k tets), written to gpurun_out/fp64_flops.json (copy to profiles/).
bench.py divides these by ITS OWN measured kernel times for the `bound: fp64` rooflines."""
import csv
import io
import json
import subprocess
import sys

METRICS = ["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
           "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "gpu__time_duration.sum"]
cmd = ["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "--csv", "-k",
       "regex:accd_kernel|elastic_state_kernel|elastic_hessian_kernel", sys.executable, "scripts/newton_ncu.py"]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
rows = list(csv.DictReader(io.StringIO(out[out.index('"ID"'):])))
per = {}
for r in rows:
    kn = r["Kernel Name"]
    name = "accd_kernel" if "accd_kernel" in kn else ("elastic_state_kernel" if "elastic_state" in kn else "elastic_hessian_kernel")
    per.setdefault((name, r["ID"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
res = {}
launches = {}
for (name, lid), m in per.items():
    launches.setdefault(name, []).append((int(lid), m))
for name, ls in launches.items():
    ls.sort(key=lambda t: t[0])
    take = ls[-2:] if name == "accd_kernel" else ls[-1:]   # one CCD filter = a VT launch + an EE launch; warm ones
    res[name] = {"flops_per_launch": sum(2 * m[METRICS[0]] + m[METRICS[1]] + m[METRICS[2]] for _, m in take),
                 "dfma": sum(m[METRICS[0]] for _, m in take), "dadd": sum(m[METRICS[1]] for _, m in take),
                 "dmul": sum(m[METRICS[2]] for _, m in take), "ncu_time_ns": sum(m[METRICS[3]] for _, m in take),
                 "launches_summed": len(take)}
# the elastic blocks are two launches (eigen phase + write-out phase): one entry for the pair
e1, e2 = res.pop("elastic_state_kernel"), res.pop("elastic_hessian_kernel")
res["elastic_blocks_kernel"] = {k: e1[k] + e2[k] for k in e1}
res["elastic_blocks_kernel"]["kernels"] = "elastic_state_kernel + elastic_hessian_kernel"
res["accd_kernel"]["workload"] = "CCD filter of cloth-stack-4x140x140, random 0.3 d_hat step (bench newton.ccd)"
res["elastic_blocks_kernel"]["workload"] = "400k random tets (bench newton.elastic)"
json.dump(res, open("gpurun_out/fp64_flops.json", "w"), indent=1)
print(json.dumps(res))
