# The last reference C3 gradient tasks on the host cores (background) while the
# GPU suite runs (2 GPUs: the NCCL / multi-device tests included).
#   gpurun --gpus 2 --timeout 3000 -- bash tools/golden_c3_rest.sh
mkdir -p gpurun_out/c3jobs3
(cd oracle && STINLA_REF=$GRAFT_REPO_ROOT/baseline/_ref PYTHONDONTWRITEBYTECODE=1 nohup python make_golden_c3.py 4 7 ../gpurun_out/c3jobs3 4,6,10,19 > ../gpurun_out/r2_golden_c3d.log 2>&1; cp ../tests/golden/c3.npz ../gpurun_out/c3_full.npz) &
GP=$!
timeout 1500 python -m pytest tests -m gpu -q -rs 2>&1 | tail -8 > gpurun_out/r2_G_pytest.log
wait $GP
