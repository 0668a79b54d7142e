# Round-2 evidence run (one GPU): the remaining reference C3 golden jobs on the
# host cores in the background; parity of the current build, POBTAF task
# profiles, an ncu launch list of the C2 step and --set full summaries of the
# top kernels in the foreground.
#   gpurun --timeout 3500 -- bash tools/profile_r02.sh
mkdir -p gpurun_out/c3jobs2 gpurun_out/ncu
(cd oracle && STINLA_REF=$GRAFT_REPO_ROOT/baseline/_ref PYTHONDONTWRITEBYTECODE=1 nohup python make_golden_c3.py 14 2 ../gpurun_out/c3jobs2 4,5,6,7,9,10,11,12,13,16,18,19,22,23 > ../gpurun_out/r2_golden_c3c.log 2>&1; cp ../tests/golden/c3.npz ../gpurun_out/c3_full.npz) &
GP=$!
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_dist.py tests/test_gpu_objective.py tests/test_gpu_pipeline.py -m gpu -q -x -rs 2>&1 | tail -6 > gpurun_out/r2_F_pytest.log
timeout 300 python tools/prof_dag.py 12 5026 3 > gpurun_out/r2_F_profdag_c3.log 2>&1
timeout 300 python tools/prof_dag.py 48 2048 6 > gpurun_out/r2_F_profdag_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu/r2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-inla > gpurun_out/ncu/r2_launches.out 2>&1
for spec in "sinv:sinv_persistent:tools/run_c2_step.py" "pobtaf_c2:pobtaf_dag:tools/run_c2_step.py" "sweep_c2:sweep_kernel:tools/run_c2_step.py"; do
  name=${spec%%:*}; rest=${spec#*:}; kre=${rest%%:*}; script=${rest#*:}
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:$kre -c 1 -o /tmp/$name python $script > gpurun_out/ncu/$name.out 2>&1
  ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/ncu/${name}_raw.csv 2>&1
  ncu -i /tmp/$name.ncu-rep --page details --csv > gpurun_out/ncu/${name}_details.csv 2>&1
done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:pobtaf_dag -c 1 -o /tmp/pobtaf_c3 python tools/run_pobtaf.py 12 5026 3 > gpurun_out/ncu/pobtaf_c3.out 2>&1
ncu -i /tmp/pobtaf_c3.ncu-rep --page raw --csv > gpurun_out/ncu/pobtaf_c3_raw.csv 2>&1
ncu -i /tmp/pobtaf_c3.ncu-rep --page details --csv > gpurun_out/ncu/pobtaf_c3_details.csv 2>&1
ls -la gpurun_out/ncu
wait $GP
