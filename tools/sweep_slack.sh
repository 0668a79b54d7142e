# POBTAF chain hand-off vs the poll back-off of the TRSM tasks off the panel
# chain (STBTA_SLACK_NS; 32 = the round-1/2 behaviour), C2 and C3-shaped.
#   gpurun --timeout 1200 -- bash tools/sweep_slack.sh
for ns in 32 1024 4096; do
  echo "== slack_ns $ns" >> gpurun_out/slack_c2.log
  STBTA_SLACK_NS=$ns timeout 200 python tools/prof_dag.py 48 2048 6 >> gpurun_out/slack_c2.log 2>&1
done
for ns in 32 1024; do
  echo "== slack_ns $ns" >> gpurun_out/slack_c3.log
  STBTA_SLACK_NS=$ns timeout 200 python tools/prof_dag.py 12 5026 3 >> gpurun_out/slack_c3.log 2>&1
done
