timeout 120 python tools/timer_skew.py > gpurun_out/r2_skew.log 2>&1
