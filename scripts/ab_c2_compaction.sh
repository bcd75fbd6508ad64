B="python bench.py --no-cpu --no-e2e --no-exact --no-configs --steps 10 --warmup 3"
for r in 1 2 3 4; do
  for v in dense level; do
    env=""; [ $v = dense ] && env="FSBM_DENSE_COMPACTION=1"
    env $env timeout 600 $B > gpurun_out/c_${v}_$r.json 2>/dev/null
    echo "$v $(grep -o '"value": [0-9.]*' gpurun_out/c_${v}_$r.json | head -1 | cut -d' ' -f2) $(grep -o '"kernel_ms": [0-9.]*' gpurun_out/c_${v}_$r.json | head -1)" >> gpurun_out/ab.txt
  done
done
