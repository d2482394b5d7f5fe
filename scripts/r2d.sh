set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/r2d_tests.log; cat gpurun_out/r2d_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo bench rc=$?
tail -c 300 gpurun_out/r2d_bench.err
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/r2d_bench.json") if l.startswith("{")][-1])
for k in ("newton", "newton_cloth_on_sphere"):
    n = d[k]
    print(k, {q: round(n[q], 4) for q in ("symbolic_ms", "assembly_numeric_ms", "spmv_ms", "pcg_solve_ms", "detect_ms")}, n["per_newton_iteration_ms"]["total"], n["newton_direction_e2e"]["ms"])
PY
python - <<'PY'
import json
d = json.loads([l for l in open("gpurun_out/r2d_bench.json") if l.startswith("{")][-1])
for k in ("newton", "newton_cloth_on_sphere"):
    print(k, "pcg_mas", json.dumps(d[k]["pcg_mas"])[:600]); print(k, "e2e mas", d[k]["newton_direction_e2e_mas"]["ms"], d[k]["newton_direction_e2e_mas"]["pcg_iters"])
PY
