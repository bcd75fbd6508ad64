#!/bin/bash
# A/B of library builds on one box: scripts/ab_variants.sh "<variants>" "<grids>" [reps]
#   variants: names of build/ab/<name>.so, or "cur" for the in-tree library
#   grids: 33 66 132 264 (264 = one GPU's 106x600x50 C5 patch)
# -> gpurun_out/ab.txt: "<variant> <nkr> <value>" lines, interleaved per repetition
vars=$1; grids=$2; reps=${3:-1}
mkdir -p gpurun_out
B="python bench.py --no-cpu --no-e2e --no-exact --no-configs --steps 3 --warmup 1"
for r in $(seq $reps); do
  for n in $grids; do
    for v in $vars; do
      case $n in
        264) g="--nkr 264 --ni 106 --nj 600 --steps 2" ;;
        33) g="" ;;
        *) g="--nkr $n" ;;
      esac
      lib=""; [ "$v" != "cur" ] && lib="FSBM_LIB_PATH=build/ab/$v.so"
      env $lib timeout 600 $B $g > gpurun_out/ab_${v}_${n}_$r.log 2>&1
      echo "$v $n $(grep -o '"value": [0-9.]*' gpurun_out/ab_${v}_${n}_$r.log | head -1 | cut -d' ' -f2) $(grep -o '"green": [a-z]*' gpurun_out/ab_${v}_${n}_$r.log | head -1)" | tee -a gpurun_out/ab.txt
    done
  done
done
