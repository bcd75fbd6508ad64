# Round-1 final evidence: GPU tests, smoke, bench lines of every config, ncu of the headline kernel
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/final_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/final_smoke.log
bash scripts/r01_all_configs.sh
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:coal_dmma_kernel -c 1 -o gpurun_out/dmma_c2_final python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_final.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu list rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coal_dmmag -c 1 -o gpurun_out/dmmag_c3_final python bench.py --nkr 66 --ni 60 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu c3 rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:coal_dmmag -c 1 -o gpurun_out/dmmag_c4_final python bench.py --nkr 132 --ni 20 --steps 1 --warmup 0 --no-e2e --no-cpu > /dev/null 2>&1; echo "ncu c4 rc=$?"
