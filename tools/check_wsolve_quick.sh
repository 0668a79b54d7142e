# quick W-solve timing + parity (C2 / C3 shapes)
timeout 300 python -m pytest tests/test_gpu_wsolve.py -m gpu -q -x 2>&1 | tail -3 > gpurun_out/r2_wq_pytest.log
for s in "48 2048 6" "48 5025 3" "48 2048 6 4"; do
  timeout 300 python tools/bench_wsolve.py $s >> gpurun_out/r2_wq_bench.jsonl 2>> gpurun_out/r2_wq_bench.err
done
