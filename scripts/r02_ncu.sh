# ncu full captures (one coal_dmma launch each) of the headline (thunderstorm) and dense C2 inputs
# usage: scripts/r02_ncu.sh <tag> [extra bench args]
tag=$1; shift
for inp in thunderstorm dense; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:coal_dmma -c 1 \
    -o gpurun_out/ncu_${tag}_${inp} python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-exact --no-configs --input $inp "$@" > gpurun_out/ncu_${tag}_${inp}.log 2>&1
  echo "$inp ncu rc=$?"
  ncu -i gpurun_out/ncu_${tag}_${inp}.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_${tag}_${inp}_src.csv 2>/dev/null
  ncu -i gpurun_out/ncu_${tag}_${inp}.ncu-rep --page raw --csv > gpurun_out/ncu_${tag}_${inp}_raw.csv 2>/dev/null
done
