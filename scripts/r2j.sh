set -u
mkdir -p gpurun_out
( time python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2j_ref.json 2> gpurun_out/r2j_ref.err ) 2>&1 | grep real
( time python bench.py > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err ) 2>&1 | grep real
python - <<'PY'
import json
r = json.loads([l for l in open("gpurun_out/r2j_ref.json") if l.startswith("{")][-1])
d = json.loads([l for l in open("gpurun_out/r2j_bench.json") if l.startswith("{")][-1])
print("ref arm:", r["value"], r["cpu_baseline"]["kind"], r["cpu_baseline"]["cores"], "port", r["c_port"]["value"])
print("b200:", d["value"], d["e2e"]["value"], d["cpu_baseline"]["value"], d.get("cpu_reference_python"))
print("ratios: e2e", d["e2e"]["value"] / r["value"], "device", d["value"] / r["value"])
print(d["fp64"].get("roofline_elastic_blocks_kernel"))
PY
