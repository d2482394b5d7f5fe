set -u
mkdir -p gpurun_out
OUT=gpurun_out/r2_sanitizer.txt
echo "# compute-sanitizer on the round-2 kernels (B200)" > $OUT
echo >> $OUT
echo "## memcheck: tests/test_gpu_symbolic.py test_gpu_mas.py test_gpu_elasticity.py" >> $OUT
timeout 2400 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_symbolic.py tests/test_gpu_mas.py tests/test_gpu_elasticity.py -x -q 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|ERROR SUMMARY|Invalid|error [0-9]" | head -30 >> $OUT
echo >> $OUT
echo "## racecheck: tests/test_gpu_symbolic.py (row-wise symbolic kernels: shared-memory sets, __syncwarp ordering)" >> $OUT
timeout 2400 compute-sanitizer --tool racecheck --print-limit 5 python -m pytest tests/test_gpu_symbolic.py -x -q -k "all-sizes or pairs-only or no-blocks or factor" 2>&1 | grep -E "COMPUTE-SANITIZER|passed|failed|RACECHECK SUMMARY|hazard" | sort | uniq -c | sort -rn | head -20 >> $OUT
cat $OUT
