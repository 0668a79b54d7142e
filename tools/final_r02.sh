# Round-2 final one-GPU evidence: smoke, the GPU suite, bench.py as the driver
# runs it (both arms).
#   gpurun --timeout 3500 -- bash tools/final_r02.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_final_smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/r2_final_pytest1.log
timeout 1500 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_final_bench1.json 2> gpurun_out/r2_final_bench1.err
timeout 1800 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_final_ref1.json 2> gpurun_out/r2_final_ref1.err
