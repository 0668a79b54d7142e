# Round-2 closing run (2 GPUs): the whole GPU suite incl. the 2-rank NCCL tests,
# smoke, and the N=1 bench line of the final build.
#   gpurun --gpus 2 --timeout 2400 -- bash tools/final_r02_b.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_close_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/r2_close_pytest2.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_close_bench1.json 2> gpurun_out/r2_close_bench1.err
