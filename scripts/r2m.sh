python -m pytest tests/test_gpu_layout.py tests/test_gpu_stencils.py tests/test_gpu_symbolic.py tests/test_gpu_solver.py -x -q 2>&1 | tail -5
python scripts/layout_probe.py stack 2>&1 | tail -4
python scripts/layout_probe.py sphere 2>&1 | tail -4
