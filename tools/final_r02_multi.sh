# Round-2 final multi-GPU evidence (4 GPUs): bench.py at N = 2 / 4 (self-launched
# torchrun) and C5 at P = 2 / 4.
#   gpurun --gpus 4 --timeout 2400 -- bash tools/final_r02_multi.sh
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2_final_bench4.json 2> gpurun_out/r2_final_bench4.err
timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r2_final_bench2.json 2> gpurun_out/r2_final_bench2.err
for g in 2 4; do timeout 300 python bench.py --config c5 --gpus $g --steps 3 --warmup 1 >> gpurun_out/r2_final_c5.jsonl 2>> gpurun_out/r2_final_c5.err; done
