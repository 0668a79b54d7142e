# ncu evidence for the consumed-barrier tile-engine build (one GPU): launch list
# of the C2 step, --set full of POBTASI / POBTAF (C2) and POBTAF at the C3 block size.
#   gpurun --timeout 1800 -- bash tools/profile_r02_cb.sh
mkdir -p gpurun_out/ncu_cb
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_cb/launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-inla > gpurun_out/ncu_cb/launches.out 2>&1
for spec in "sinv:sinv_persistent:tools/run_c2_step.py" "pobtaf_c2:pobtaf_dag:tools/run_c2_step.py"; do
  name=${spec%%:*}; rest=${spec#*:}; kre=${rest%%:*}; script=${rest#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$kre -c 1 -o /tmp/$name python $script > gpurun_out/ncu_cb/$name.out 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/ncu_cb/${name}_raw.csv 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pobtaf_dag -c 1 -o /tmp/pobtaf_c3 python tools/run_pobtaf.py 12 5026 3 > gpurun_out/ncu_cb/pobtaf_c3.out 2>&1
ncu -i /tmp/pobtaf_c3.ncu-rep --page raw --csv > gpurun_out/ncu_cb/pobtaf_c3_raw.csv 2>&1
ls -la gpurun_out/ncu_cb
