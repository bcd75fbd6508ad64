# A/B of the FAST compaction: dense CUB select vs the level-major padded list (default)
B="python bench.py --no-cpu --no-e2e --no-exact --no-configs --steps 5 --warmup 2"
for r in 1 2; do
for cfg in "c2:" "cf03:--cf 0.3" "n66:--nkr 66" "n264:--nkr 264 --ni 106 --nj 600 --steps 2"; do
  name=${cfg%%:*}; args=${cfg#*:}
  for v in dense level; do
    env=""; [ $v = dense ] && env="FSBM_DENSE_COMPACTION=1"
    env $env timeout 600 $B $args > gpurun_out/l_${v}_${name}.json 2>/dev/null
    echo "$v $name $(grep -o '"value": [0-9.]*' gpurun_out/l_${v}_${name}.json | head -1 | cut -d' ' -f2) $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/l_${v}_${name}.json | head -1)" >> gpurun_out/ab.txt
  done
done; done
