# POBTAF chunk / look-ahead / remainder sweep at the C3 block size and C2
# (STBTA_CHUNK / STBTA_LOOK / STBTA_REMAINDER override the defaults).
#   gpurun --timeout 1500 -- bash tools/sweep_pobtaf.sh
out=gpurun_out/r2_sweep_pobtaf.log
: > $out
for cfg in "8 2 1" "8 2 0" "6 2 1" "12 2 1" "16 2 1" "8 3 1" "4 2 1"; do
  set -- $cfg
  echo "C3shape chunk=$1 look=$2 rem=$3 $(STBTA_CHUNK=$1 STBTA_LOOK=$2 STBTA_REMAINDER=$3 timeout 300 python tools/prof_dag.py 12 5026 3 2>&1 | sed -n 2p)" >> $out
done
for cfg in "4 3 0" "4 3 1" "8 3 0" "4 2 0" "6 3 0"; do
  set -- $cfg
  echo "C2 chunk=$1 look=$2 rem=$3 $(STBTA_CHUNK=$1 STBTA_LOOK=$2 STBTA_REMAINDER=$3 timeout 300 python tools/prof_dag.py 48 2048 6 2>&1 | sed -n 2p)" >> $out
done
cat $out
