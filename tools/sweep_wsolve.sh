# W-solve parameter sweep / phase profile at the C2 and C3 shapes
export BW_QUICK=1 BW_PROF=1 STBTA_WS_COLMAP=1
for s in "48 2048 6" "48 5025 3"; do
  for cu in "64 16" "64 32" "32 32" "128 32"; do
    set -- $cu
    STBTA_WS_CHUNK=$1 STBTA_WS_U=$2 timeout 200 python tools/bench_wsolve.py $s >> gpurun_out/r2_wsweep.jsonl 2>> gpurun_out/r2_wsweep.err
  done
done
