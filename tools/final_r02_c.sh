# Round-2 closing run on the final build (2 GPUs): smoke, the whole GPU suite
# incl. the 2-rank NCCL tests, bench lines at N=1 and N=2, the reference arm.
#   gpurun --gpus 2 --timeout 3000 -- bash tools/final_r02_c.sh
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_end_smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/r2_end_pytest2.log
CUDA_VISIBLE_DEVICES=0 timeout 1200 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2_end_bench1.json 2> gpurun_out/r2_end_bench1.err
timeout 1200 python bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r2_end_bench2.json 2> gpurun_out/r2_end_bench2.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_end_ref1.json 2> gpurun_out/r2_end_ref1.err
