# ncu evidence for the C2 step with the shared-W solve: launch list of the
# bench step and a --set full capture of the W-based POBTAS kernel.
#   gpurun --timeout 1800 -- bash tools/profile_wsolve.sh
mkdir -p gpurun_out/ncu
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/r2w_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-inla > gpurun_out/ncu/r2w_launches.out 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:wsolve -c 1 -o /tmp/wsolve_c2 python tools/run_c2_step.py > gpurun_out/ncu/wsolve_c2.out 2>&1
ncu -i /tmp/wsolve_c2.ncu-rep --page raw --csv > gpurun_out/ncu/wsolve_c2_raw.csv 2>&1
ncu -i /tmp/wsolve_c2.ncu-rep --page details --csv > gpurun_out/ncu/wsolve_c2_details.csv 2>&1
ls -la gpurun_out/ncu
