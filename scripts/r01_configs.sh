# Round-1 measurements of the non-headline BASELINE configs (C3/C4/C5 patch) + dmmag ncu
set -x
python bench.py --nkr 66 --steps 5 --warmup 3 --e2e-steps 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --nkr 132 --steps 3 --warmup 3 --no-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --nkr 264 --ni 106 --nj 600 --steps 3 --warmup 3 --no-e2e --cpu-seconds 20 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coal_dmmag -c 1 -o gpurun_out/dmmag_c3 python bench.py --nkr 66 --ni 60 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coal_dmmag -c 1 -o gpurun_out/dmmag_c4 python bench.py --nkr 132 --ni 20 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c3.csv python bench.py --nkr 66 --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
tail -c 2000 gpurun_out/bench_c3.json gpurun_out/bench_c4.json gpurun_out/bench_c5.json | cut -c1-400
