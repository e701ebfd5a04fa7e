#!/bin/bash
# compute-sanitizer gates over the small GPU parity cases: every
# librs kernel of the dense and all-communities paths, the getters and top-K.
# Usage (GPU box): bash tools/sanitize.sh [outdir]
OUT=${1:-gpurun_out/san}
mkdir -p "$OUT"
SEL="worked_example or karate or triad_counts_right or degenerate or many_columns or uncoded or (rsgen_scaled and orkut-0.003) or topk_edges or complete_graphs_all"
: > "$OUT/summary.txt"
for tool in memcheck initcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 100 --error-exitcode 99 \
      python -m pytest -x -q -p no:cacheprovider tests/test_gpu_parity.py tests/test_gpu_sparse.py -k "$SEL" > "$OUT/$tool.log" 2>&1
  rc=$?
  nerr=$(grep -c "========= " "$OUT/$tool.log")
  summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$OUT/$tool.log" | tail -1)
  echo "$tool rc=$rc lines=$nerr $summ" >> "$OUT/summary.txt"
done
cat "$OUT/summary.txt"
