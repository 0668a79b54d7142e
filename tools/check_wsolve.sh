# W-based POBTAS: parity tests, timings against the tile sweeps, smoke and the N=1 bench line.
#   gpurun --timeout 2400 -- bash tools/check_wsolve.sh
timeout 900 python -m pytest tests/test_gpu_wsolve.py tests/test_gpu_solver.py tests/test_gpu_pipeline.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2_wsolve_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_wsolve_smoke.log 2>&1
for s in "48 2048 6" "48 5025 3" "48 2048 6 4"; do
  BW_PROF=1 timeout 300 python tools/bench_wsolve.py $s >> gpurun_out/r2_wsolve_bench.jsonl 2>> gpurun_out/r2_wsolve_bench.err
done
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_wsolve_bench1.json 2> gpurun_out/r2_wsolve_bench1.err
timeout 600 python bench.py --no-inla --no-cpu --steps 20 --warmup 5 --solve tile > gpurun_out/r2_wsolve_bench1_tile.json 2>> gpurun_out/r2_wsolve_bench1.err
