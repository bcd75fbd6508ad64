#!/bin/bash
# ncu --set full captures (one launch each, source-attributed) of the coalescence kernels:
#   dmma  (C2, 33 bins)          dmmag66 (C3 slab, 66 bins)    dmmag264 (C5 slab, 264 bins)
# usage (GPU box): scripts/ncu_kernels.sh <tag> [cases...]   -> gpurun_out/ncu_<tag>_<case>.*
tag=$1; shift
cases=${*:-"dmma dmmag66 dmmag264"}
B="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-exact --no-configs"
for c in $cases; do
  case $c in
    dmma)     k=coal_dmma_kernel; args="" ;;
    dmmag66)  k=coal_dmmag;       args="--nkr 66 --ni 60" ;;
    dmmag132) k=coal_dmmag;       args="--nkr 132 --ni 20" ;;
    dmmag264) k=coal_dmmag;       args="--nkr 264 --ni 4 --nj 600" ;;
  esac
  o=gpurun_out/ncu_${tag}_${c}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:$k -c 1 -o $o $B $args > $o.log 2>&1
  echo "$c ncu rc=$?"
  ncu -i $o.ncu-rep --page source --csv --print-source cuda,sass > ${o}_src.csv 2>/dev/null
  python scripts/ncu_summary.py report $o.ncu-rep ${o}_summary.json > /dev/null 2>&1
  python scripts/ncu_sass_hot.py ${o}_src.csv 50 > ${o}_hot.txt 2>&1
  # keep the merge-back small: the report and source page stay on the box unless asked for
  [ -z "$KEEP_REP" ] && rm -f $o.ncu-rep
  gzip -f ${o}_src.csv
done
