# Round-2 closing multi-GPU evidence on the final build (4 GPUs):
# the 4-GPU NCCL test, bench.py at N = 4 (self-launched ranks), C5 at P = 2 / 4.
#   gpurun --gpus 4 --timeout 2400 -- bash tools/final_r02_multi2.sh
timeout 600 python -m pytest tests/test_gpu_nccl.py -m gpu -q -rs 2>&1 | tail -4 > gpurun_out/r2i_nccl4.log
timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r2i_bench4.json 2> gpurun_out/r2i_bench4.err
for g in 2 4; do timeout 300 python bench.py --config c5 --gpus $g --steps 3 --warmup 1 >> gpurun_out/r2i_c5.jsonl 2>> gpurun_out/r2i_c5.err; done
