"""Regenerate the 'Round 2 at a glance' table of profiles/README.md from the bench lines of one tag.

    python scripts/profiles_readme.py r2l
"""
import json
import re
import sys

tag = sys.argv[1]
d = json.load(open(f"profiles/{tag}_bench.json"))
r = json.load(open(f"profiles/{tag}_bench_reference_arm.json"))
n, sph = d["newton"], d["newton_cloth_on_sphere"]
m1, m2 = n["pcg_mas"]["levels_1"], n["pcg_mas"]["levels_2"]
vs = n["vs_reference_cpu"]
ref_solve = r["newton"]["cloth_stack"].get("reference_pcg_solve") or {}
steps = ", ".join(f"{st['wall_ms']:.0f} ms ({st['newton_iters']} Newton / {st['pcg_iters']} PCG)" for st in n["time_step"]["steps"])
rows = [
    ("PSD barrier Hessian stencils/s (1 M near-parallel EE, dense blocks)", "4.09 - 4.14 G/s",
     f"**{d['value']/1e9:.2f} G/s**, {d['roofline']['achieved']:.0f} GB/s = **{d['roofline']['frac']:.3f}** of the measured HBM peak, "
     f"DRAM traffic {d['roofline']['traffic']/d['roofline']['algorithmic_bytes_per_step']:.3f} x algorithmic"),
    ("e2e strict (host in -> every dense block back on the host) vs the reference arm proper (the unmodified `tetipc` package, "
     f"{r['cpu_baseline']['cores']} processes)", "--",
     f"{d['e2e']['value']/1e6:.1f} M/s vs **{r['value']/1e6:.2f} M/s** = {d['e2e']['value']/r['value']:.0f} x (device-resident: "
     f"{d['value']/r['value']:.0f} x); one reference process: {r['cpu_baseline'].get('one_process', 0)/1e3:.1f} k/s"),
    ("same vs the C port of the reference path on the same table (`c_port`, all host threads)", "41.5 - 44.5 M/s vs 33 - 40 M/s (250 k table)",
     f"{d['e2e']['value']/1e6:.1f} M/s vs {r['c_port']['value']/1e6:.1f} M/s (PCIe-bound: 1.25 GB back per step)"),
    ("symbolic assembly, 1.03 M contacts", "1.27 ms (global sort of 16.5 M slots)", f"**{n['symbolic_ms']:.2f} ms** (row-wise, bitwise the same matrices)"),
    ("numeric assembly (dense) / from factors / SpMV", "0.298 / 0.287 / 0.0275 ms",
     f"{n['assembly_numeric_ms']:.3f} / {n['fused']['assembly_from_factors_ms']:.3f} / {n['spmv_ms']:.4f} ms "
     f"({n['roofline_assembly']['frac']:.2f} / {n['roofline_assembly_factors']['frac']:.2f} / {n['roofline_spmv']['frac']:.2f} of HBM)"),
    ("assembly + SpMV a Newton iteration pays (symbolic + numeric from factors + SpMV)", "1.59 ms", f"**{n['per_newton_iteration_ms']['total']:.2f} ms**"),
    ("PCG per iteration, block-Jacobi", "34 - 38 us", f"**{n['pcg_ms_per_iter']*1e3:.1f} us** (L2 eviction hints, 27-row chunks)"),
    ("PCG to 1e-4, block-Jacobi", "244 iterations, 9.0 - 9.2 ms", f"{n['pcg_iters']} iterations, {n['pcg_solve_ms']:.2f} ms"),
    ("PCG to 1e-4 (same stopping rule), MAS preconditioner, 1 level", "--",
     f"**{m1['iters']} iterations, {m1['setup_ms']:.2f} ms setup + {m1['solve_ms']:.2f} ms solve = {m1['setup_plus_solve_ms']:.2f} ms** "
     f"({m1['us_per_iter']:.1f} us per iteration; order {n['pcg_mas']['order_ms']:.2f} ms once per time step)"),
    ("same, 2 levels", "--", f"{m2['iters']} iterations, {m2['setup_plus_solve_ms']:.2f} ms (the coarse level does not pay on a contact-only matrix, DESIGN 4.8)"),
    ("`pcg_solve` to 1e-4: the unmodified `tetipc.solver.pcg_solve` (compiled `_core` backend, one process) on this host", "--",
     f"**{ref_solve.get('ms', 0)/1e3:.1f} s, {ref_solve.get('iters')} iterations** vs {n['pcg_solve_ms']:.1f} ms, {n['pcg_iters']} iterations here "
     f"(block-Jacobi: {vs.get('pcg_solve') or 0:.0f} x) and {m1['setup_plus_solve_ms']:.1f} ms (MAS: {vs.get('pcg_solve_vs_mas') or 0:.0f} x)"),
    ("Newton direction end to end (host x in -> host d out)", "12.9 ms",
     f"{n['newton_direction_e2e']['ms']:.1f} ms (block-Jacobi), **{n['newton_direction_e2e_mas']['ms']:.1f} ms** (MAS); "
     f"the reference's way on this host (C-port blocks + `_core.matvec_blocks` PCG, projected): {vs['newton_direction']:.0f} x slower"),
    ("cloth on sphere (configs[2]: 110 k vertices, 273 k contacts): symbolic / numeric / SpMV / direction e2e", "0.54 / 0.057 / 0.015 / 3.7 ms (start of round 2)",
     f"{sph['symbolic_ms']:.2f} / {sph['assembly_numeric_ms']:.3f} / {sph['spmv_ms']:.3f} / {sph['newton_direction_e2e']['ms']:.1f} ms "
     f"(block-Jacobi needs {sph['pcg_iters']} iterations there: MAS is a loss, {sph['pcg_mas']['levels_1']['setup_plus_solve_ms']:.2f} vs {sph['pcg_solve_ms']:.2f} ms)"),
    ("elasticity, 400 k tets (energy + gradient + projected 12x12)", "0.433 ms", f"**{n['elastic']['blocks_ms']:.3f} ms** (two phases)"),
    (f"fp64 rooflines (`bound: \"fp64\"`, peak {d['fp64']['fp64_tflops_measured']:.1f} TFLOP/s measured)", "--",
     f"`accd_kernel` {d['fp64']['roofline_accd_kernel']['frac']:.3f}, elastic pair {d['fp64']['roofline_elastic_blocks_kernel']['frac']:.3f} "
     "(latency-bound Jacobi / ACCD iterations, not throughput)"),
    ("detect (broad + narrow)", "0.77 + 0.58 ms", f"{n['broad_phase_ms']:.2f} + {n['narrow_phase_ms']:.2f} ms"),
    ("CCD: swept candidates + ACCD filter", "0.89 ms", f"{n['ccd']['sweep_plus_filter_ms']:.2f} ms"),
    ("whole time steps (`stepper.advance_time_step`, soft cloth stack)", "25 - 35 ms (7 - 8 Newton iterations); first step 240 - 310 ms",
     steps + " -- one swept join per Newton iteration instead of two (DESIGN 4.7); wall clock incl. every host sync"),
]
table = "| quantity | round 1 (r1h) | round 2 (" + tag + ") |\n|---|---|---|\n" + "\n".join(f"| {a} | {b} | {c} |" for a, b, c in rows) + "\n"
p = "profiles/README.md"
s = open(p).read()
s = re.sub(r"<!-- glance:begin -->.*?<!-- glance:end -->", "<!-- glance:begin -->\n" + table + "<!-- glance:end -->", s, flags=re.S)
open(p, "w").write(s)
print(table)
