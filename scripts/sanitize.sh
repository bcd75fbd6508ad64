#!/bin/bash
# compute-sanitizer over one small step per kernel (scripts/sanitize_cases.py).
# Usage (on the GPU box): scripts/sanitize.sh [out_dir]   -> <out_dir>/<tool>_<case>.txt + summary.txt
OUT=${1:-gpurun_out/sanitizer}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
CASES="dmma dmmag66 dmmag264 direct exact host group stiff moments"
: > "$OUT/summary.txt"
for tool in memcheck racecheck synccheck initcheck; do
  for c in $CASES; do
    f="$OUT/${tool}_${c}.txt"
    extra=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report all"
    timeout 900 $CS --tool $tool $extra \
      --print-limit 20 python scripts/sanitize_cases.py $c > "$f" 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|Error" "$f" | tail -2 | tr '\n' ' ')
    ok=$(grep -c "sanitize case $c: ok" "$f")
    echo "$tool $c rc=$rc case_ok=$ok :: $summ" | tee -a "$OUT/summary.txt"
  done
done
