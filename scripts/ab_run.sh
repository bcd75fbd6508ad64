# A/B bench runs of library variants built by scripts/build_variant.sh (one box, interleaved)
rm -f gpurun_out/ab.txt
for rep in 1 2; do
for spec in "$@"; do
  v=${spec%%:*}; envs=${spec#*:}; [ "$envs" = "$spec" ] && envs=""
  env $envs FSBM_LIB_PATH=build/ab/$v.so timeout 200 python bench.py --no-cpu --no-e2e --no-exact --no-configs --steps 10 > gpurun_out/b_$v.log 2>&1
  echo "$spec $(grep -o '"value": [0-9.]*' gpurun_out/b_$v.log | head -1)" >> gpurun_out/ab.txt
done; done
