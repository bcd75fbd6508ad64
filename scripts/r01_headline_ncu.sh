# ncu evidence for the headline (C2, 33 bins, coal_dmma): full capture of one launch + launch list
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:coal_dmma_kernel -c 1 -o gpurun_out/dmma_c2_tmem python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1; echo full=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo list=$?
