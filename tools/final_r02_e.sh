# Round-2 closing evidence on the final build (C-tile prefetch, per-strip POTRF load) (2 GPUs):
# smoke, the whole GPU suite (incl. the 2-rank NCCL tests), bench.py at N = 1 / 2,
# and the UPDATE tile-engine micro-benchmark.
#   gpurun --gpus 2 --timeout 2400 -- bash tools/final_r02_e.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2h_smoke.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/r2h_pytest2.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2h_bench1.json 2> gpurun_out/r2h_bench1.err
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2h_bench2.json 2> gpurun_out/r2h_bench2.err
