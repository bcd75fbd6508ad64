#!/bin/bash
# compute-sanitizer over one small step per kernel (scripts/sanitize_cases.py).
# Usage (on the GPU box): scripts/sanitize.sh [out_dir]   -> <out_dir>/<tool>_<case>.txt + summary.txt
#  * racecheck runs in analysis mode: hazards are aggregated per (access, access) site pair,
#    so the summary lists every distinct racing pair of source lines.
#  * synccheck (CUDA 12.9) aborts any tcgen05 kernel that initialises no mbarrier ("Missing
#    init" at shared 0x0, reported outside the kernel body); coal_dmmag has none, so synccheck
#    runs on a build with -DFSBM_SYNCCHECK_MBAR (one unused mbarrier, otherwise identical).
OUT=${1:-gpurun_out/sanitizer}
mkdir -p "$OUT"
CS=/usr/local/cuda/bin/compute-sanitizer
CASES=${CASES:-"dmma dmmag66 dmmag264 direct exact host group stiff moments"}
SC_LIB=build/ab/synccheck.so
[ -f $SC_LIB ] || bash scripts/build_variant.sh synccheck paper_2409_07232_b200/csrc -DFSBM_SYNCCHECK_MBAR > /dev/null 2>&1
: > "$OUT/summary.txt"
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  for c in $CASES; do
    f="$OUT/${tool}_${c}.txt"
    extra=""; envs=""
    [ "$tool" = "memcheck" ] && extra="--leak-check no"
    [ "$tool" = "racecheck" ] && extra="--racecheck-report analysis"
    [ "$tool" = "synccheck" ] && envs="FSBM_LIB_PATH=$SC_LIB"
    env $envs timeout 900 $CS --tool $tool $extra --print-limit 1000 python scripts/sanitize_cases.py $c > "$f" 2>&1
    rc=$?
    summ=$(grep -E "ERROR SUMMARY|RACECHECK SUMMARY" "$f" | tail -1 | tr '\n' ' ')
    ok=$(grep -c "sanitize case $c: ok" "$f")
    echo "$tool $c rc=$rc case_ok=$ok :: $summ" | tee -a "$OUT/summary.txt"
    if [ "$tool" = "racecheck" ]; then # distinct racing site pairs
      grep -E "Race reported between|^=========     (Read|Write|Atomic)" "$f" | sed -E 's/\+0x[0-9a-f]+//; s/ at 0x[0-9a-f]+//' \
        | sort | uniq -c | sort -rn | head -12 | sed 's/^/    /' >> "$OUT/summary.txt"
    fi
  done
done
