set -u
mkdir -p gpurun_out
python -m pytest tests/test_gpu_stencils.py -q -k k2 2>&1 | tail -5
python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench rc=$?
tail -c 600 gpurun_out/r2b_bench.err
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2b_ref.json 2> gpurun_out/r2b_ref.err; echo ref rc=$?
python scripts/fp64_flops.py > gpurun_out/r2b_fp64.log 2>&1; tail -3 gpurun_out/r2b_fp64.log | cut -c1-600
