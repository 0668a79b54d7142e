# Multi-GPU evidence on one box (run under gpurun --gpus 4).
set -x
cd /root/repo
T="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1 --master-port 29512"
rm -f gpurun_out/c5_4gpu.jsonl
for N in 1 2 4; do
  $T --nproc-per-node $N bench.py --config c5 --gpus $N --steps 2 --warmup 1 2>/dev/null | grep '^{' >> gpurun_out/c5_4gpu.jsonl
done
$T --nproc-per-node 4 bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu --no-inla 2>/dev/null | grep '^{' > gpurun_out/c2_4gpu.json
python tools/bench_inla.py c4 1 2>&1 | tail -1 > gpurun_out/c4_4gpu.json
python tools/bench_inla.py c3iter 3 2>&1 | tail -1 > gpurun_out/c3iter_4gpu.json
