# POBTAF panel-chain timeline at C2
for ns in 32 34; do
echo "== $ns" >> gpurun_out/r2_chain_c2.log
STBTA_SPIN_NS=$ns timeout 300 python tools/prof_dag.py 48 2048 6 >> gpurun_out/r2_chain_c2.log 2>&1
done
