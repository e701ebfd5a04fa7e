# A/B of experiment builds on the all-communities mode (LJ shape, 10 000 communities)
for L in "$@"; do
  echo "== $L"; RS_LIBRARY=paper_2508_01485_b200/$L timeout 300 python tools/sparse_time.py lj 10000 2>&1 | grep "^all"
done
