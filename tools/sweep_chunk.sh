set -e
cd /root/repo/paper_2507_06938_b200/csrc
for cfg in "2 8 4" "3 8 4" "2 16 8" "1 8 4"; do
  set -- $cfg
  sed -i "s/^constexpr int LOOK = .*;/constexpr int LOOK = $1;/" pobtaf.cu
  sed -i "s/^STBTA_DEV int chunk_k(const Band\& g) { return g.nbt >= 24 ? [0-9]* : [0-9]*; }/STBTA_DEV int chunk_k(const Band\& g) { return g.nbt >= 24 ? $2 : $3; }/" pobtaf.cu
  grep -n "^constexpr int LOOK\|^STBTA_DEV int chunk_k" pobtaf.cu | tr '\n' ' '; echo
  make -s 2>&1 | grep -i error || true
  cd /root/repo
  python tools/prof_dag.py 48 2048 6 2>&1 | sed -n 2p
  python tools/prof_dag.py 16 5026 3 2>&1 | sed -n 2p
  cd /root/repo/paper_2507_06938_b200/csrc
done
