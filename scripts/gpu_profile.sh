#!/bin/bash
# Run on the GPU box (via gpurun): launch list of bench.py + full ncu captures of the hot kernels.
# Usage: scripts/gpu_profile.sh <tag>
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
# 1. every launch of the default bench command with its device time (cold-cache, serialised: compare shares)
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 5 --warmup 3 --skip-cpu > gpurun_out/launches_${TAG}.log 2>&1
python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
# 2. the headline kernel, full set, two launches after warm-up
ncu --set full --clock-control none --import-source on -k regex:barrier_stencil_kernel -s 4 -c 2 \
    -o gpurun_out/prof_stencil_${TAG} -f python bench.py --steps 2 --warmup 3 --skip-newton --skip-cpu \
    > gpurun_out/prof_stencil_${TAG}.log 2>&1
# 3. Newton-step kernels at bench scale
ncu --set full --clock-control none \
    -k regex:"bsr_spmv_stream_kernel|assemble_rows_kernel|assemble_numeric_kernel|assemble_factors_kernel|assemble_numeric_trio_kernel|assemble_factors_trio_kernel|scatter_gradient_kernel|block_jacobi_kernel|pcg_stream_kernel|pcg_mas_kernel|mas_setup_kernel|apply_level0_kernel|row_emit_small_kernel|row_emit_large_kernel|row_pack_kernel|join_kernel|narrow_classify_kernel|narrow_ties_kernel|accd_kernel|friction_blocks_kernel|friction_state_kernel|elastic_state_kernel|elastic_hessian_kernel" \
    -c 90 -o gpurun_out/prof_newton_${TAG} -f python scripts/newton_ncu.py --pcg > gpurun_out/prof_newton_${TAG}.log 2>&1
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_${TAG}_ref.json 2>/dev/null
python scripts/fp64_flops.py > gpurun_out/fp64_flops_${TAG}.log 2>&1
cp gpurun_out/fp64_flops.json profiles/fp64_flops.json
# 4. summarise on the box (the raw reports exceed what gpurun brings back) and ship the summaries
python scripts/summarise_profiles.py ${TAG} ${TAG} > gpurun_out/summarise_${TAG}.log 2>&1
mkdir -p gpurun_out/profiles_${TAG} && cp profiles/${TAG}_* profiles/stencil_traffic.json profiles/fp64_flops.json gpurun_out/profiles_${TAG}/
rm -f gpurun_out/prof_newton_${TAG}.ncu-rep
ls -la gpurun_out gpurun_out/profiles_${TAG} | tail -20
