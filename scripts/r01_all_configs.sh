# Round-1 bench lines for every BASELINE config on one B200 (C2 headline + C3/C4/C5 patch)
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --nkr 66 --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --nkr 132 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --nkr 264 --ni 106 --nj 600 --steps 3 --warmup 3 --no-e2e --cpu-seconds 20 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for c in c2 c3 c4 c5 ref; do python -c "
import json;d=json.load(open('gpurun_out/bench_$c.json'));r=d.get('roofline') or {};e=d.get('e2e') or {}
print('$c', round(d['value']/1e6,3), 'M', r.get('kernel'), round(r.get('frac',0),3), 'e2e', e.get('value') and round(e['value']/1e6,3), d.get('clocks'))"; done
