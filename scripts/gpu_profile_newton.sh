#!/bin/bash
# Full-scale ncu capture of the Newton-step kernels (assembly variants, SpMV, gradient, PCG).
TAG=${1:-r1}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on \
    -k regex:'assemble_rows_kernel|assemble_numeric_kernel|bsr_spmv_kernel|scatter_gradient_kernel' -s 8 -c 8 \
    -o gpurun_out/prof_newton_${TAG} -f python bench.py --steps 3 --warmup 3 --skip-cpu --n-stencils 20000 \
    > gpurun_out/prof_newton_${TAG}.log 2>&1
tail -3 gpurun_out/prof_newton_${TAG}.log
