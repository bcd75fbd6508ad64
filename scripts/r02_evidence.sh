#!/bin/bash
# Round-2 evidence on one box: -m gpu tests, smoke, the default bench line (all configs,
# parity, cpu_baseline, e2e), the launch list of the headline command, ncu of the headline
# kernel.  Outputs under gpurun_out/ (summaries small enough to merge back).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-exact --no-configs > /dev/null 2>&1
python scripts/ncu_summary.py launches gpurun_out/launches_c2.csv gpurun_out/launches_c2.json > /dev/null 2>&1
rm -f gpurun_out/launches_c2.csv
bash scripts/ncu_kernels.sh final dmma
