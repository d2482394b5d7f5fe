#!/bin/bash
# Run on the GPU box (via gpurun): launch list + full ncu capture of the stencil kernel for bench.py's workload.
# Usage: scripts/gpu_profile.sh <tag>
set -u
TAG=${1:-r1}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --skip-cpu > gpurun_out/launches_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:barrier_stencil_kernel -s 4 -c 2 \
    -o gpurun_out/prof_stencil_${TAG} -f python bench.py --steps 1 --warmup 3 --skip-newton --skip-cpu \
    > gpurun_out/prof_stencil_${TAG}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'assemble_numeric|bsr_spmv|pcg_kernel|scatter_gradient' -c 8 \
    -o gpurun_out/prof_newton_${TAG} -f python bench.py --steps 2 --warmup 3 --skip-cpu --n-stencils 20000 \
    > gpurun_out/prof_newton_${TAG}.log 2>&1
ls -la gpurun_out
