rm -f gpurun_out/ab66.txt
for v in base fz; do
  for n in 66 132; do
  FSBM_LIB_PATH=build/ab/$v.so timeout 300 python bench.py --no-cpu --no-e2e --nkr $n --steps 2 --warmup 1 > gpurun_out/b_${v}_$n.log 2>&1
  echo "$v $n $(grep -o '"value": [0-9.]*' gpurun_out/b_${v}_$n.log | head -1)" >> gpurun_out/ab66.txt
done; done
