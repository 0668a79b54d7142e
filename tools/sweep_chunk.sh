# Sweep the chunked-update parameters (look >= 2 always).
set -e
cd /root/repo/paper_2507_06938_b200/csrc
cp pobtaf.cu /tmp/pobtaf_orig.cu
for cfg in "2 3 8 4" "2 2 8 4" "2 3 8 6" "2 2 8 8" "2 3 8 2"; do
  set -- $cfg
  cp /tmp/pobtaf_orig.cu pobtaf.cu
  sed -i "s/^STBTA_DEV int look(const Band\& g) { return g.nbt >= 24 ? [0-9]* : [0-9]*; }/STBTA_DEV int look(const Band\& g) { return g.nbt >= 24 ? $1 : $2; }/" pobtaf.cu
  sed -i "s/^STBTA_DEV int chunk_k(const Band\& g) { return g.nbt >= 24 ? [0-9]* : [0-9]*; }/STBTA_DEV int chunk_k(const Band\& g) { return g.nbt >= 24 ? $3 : $4; }/" pobtaf.cu
  grep "^STBTA_DEV int look\|^STBTA_DEV int chunk_k" pobtaf.cu | tr '\n' ' '; echo
  make -s 2>&1 | grep -i error || true
  cd /root/repo
  timeout 120 python tools/prof_dag.py 48 2048 6 2>&1 | sed -n 2p
  true
  cd /root/repo/paper_2507_06938_b200/csrc
done
cp /tmp/pobtaf_orig.cu pobtaf.cu
