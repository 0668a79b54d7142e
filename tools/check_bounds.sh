# Bounds-checked runs (compute-sanitizer is closed on this pool): every kernel
# of the product through the checked build (make check -> libstbta_check.so,
# device asserts on tile / storage addressing), on small and medium shapes
# against the oracle, plus the solver / partitioned / objective GPU tests.
#   gpurun --timeout 1800 -- bash tools/check_bounds.sh
export STBTA_LIB=$PWD/paper_2507_06938_b200/libstbta_check.so
timeout 900 python tools/sanitize_cases.py medium > gpurun_out/r2_check_cases.log 2>&1; echo "rc=$?" >> gpurun_out/r2_check_cases.log
timeout 1200 python -m pytest tests/test_gpu_solver.py tests/test_gpu_dist.py tests/test_gpu_objective.py tests/test_gpu_pipeline.py tests/test_gpu_baseline_configs.py -m gpu -q -rs 2>&1 | tail -6 > gpurun_out/r2_check_pytest.log
