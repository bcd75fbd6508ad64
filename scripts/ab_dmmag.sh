# A/B timings of coal_dmmag variants (env knobs read at context creation); NKR selects the grid
for v in ${VARIANTS:-"X=1" "FSBM_DMMAG_WARPS=12" "FSBM_DMMAG_NOSKIP=1" "FSBM_FAST_KERNEL=direct"}; do
  env $v timeout 300 python bench.py --nkr ${NKR:-66} --steps 3 --warmup 1 --no-e2e --no-cpu > /tmp/ab.json 2>/tmp/ab.err || tail -3 /tmp/ab.err
  echo "nkr ${NKR:-66} $v $(python -c "import json;d=json.load(open('/tmp/ab.json'));print(round(d['value']/1e6,3),'M upd/s', round(d['roofline']['frac'],4))")"
done
