# Validate a POBTAF change: solver parity, task profiles at C2 / the C3 block size, C2 bench line.
#   gpurun --timeout 1800 -- bash tools/check_potrf.sh
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_baseline_configs.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2_J_pytest.log
timeout 300 python tools/prof_dag.py 48 2048 6 > gpurun_out/r2_J_profdag_c2.log 2>&1
timeout 300 python tools/prof_dag.py 12 5026 3 > gpurun_out/r2_J_profdag_c3.log 2>&1
timeout 900 python bench.py --no-cpu --no-inla --steps 10 --warmup 3 > gpurun_out/r2_J_bench.json 2> gpurun_out/r2_J_bench.err
