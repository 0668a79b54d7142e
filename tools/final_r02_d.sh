# Round-2 closing run (4 GPUs): bench line at N=4 (C2 replicas + C3
# iterations) and the C5 distributed solver at P=4; plus the marginal tests
# of the final build.
#   gpurun --gpus 4 --timeout 2400 -- bash tools/final_r02_d.sh
timeout 600 python -m pytest tests/test_gpu_objective.py tests/test_gpu_baseline_configs.py tests/test_gpu_wsolve.py -m gpu -q -rs 2>&1 | tail -4 > gpurun_out/r2_end_pytest_marg.log
timeout 1200 python bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r2_end_bench4.json 2> gpurun_out/r2_end_bench4.err
timeout 900 python bench.py --config c5 --gpus 4 --steps 3 --warmup 2 > gpurun_out/r2_end_c5_4.json 2> gpurun_out/r2_end_c5_4.err
