# Validate a POBTAS change: solver / partitioned / objective parity and the sweep profile.
#   gpurun --timeout 1800 -- bash tools/check_pobtas.sh
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_dist.py tests/test_gpu_objective.py tests/test_gpu_pipeline.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2_K_pytest.log
timeout 300 python tools/prof_solve.py 48 2048 6 > gpurun_out/r2_K_profsolve_c2.log 2>&1
timeout 300 python tools/prof_solve.py 12 5026 3 > gpurun_out/r2_K_profsolve_c3.log 2>&1
timeout 300 python tools/prof_solve.py 6 130 2 > gpurun_out/r2_K_profsolve_small.log 2>&1
