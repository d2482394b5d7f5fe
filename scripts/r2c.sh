set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r2c_tests.log; cat gpurun_out/r2c_tests.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench.json 2> gpurun_out/r2c_bench.err; echo bench rc=$?
tail -c 800 gpurun_out/r2c_bench.err
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2c_ref.json 2> gpurun_out/r2c_ref.err; echo ref rc=$?
tail -c 400 gpurun_out/r2c_ref.err
python scripts/fp64_flops.py > gpurun_out/r2c_fp64.log 2>&1; tail -3 gpurun_out/r2c_fp64.log | cut -c1-600
