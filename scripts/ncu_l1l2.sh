#!/bin/bash
# L1 / L2 traffic of coal_dmmag for several library builds (FSBM_LIB_PATH variants):
#   scripts/ncu_l1l2.sh "<variants>" <nkr> [bench args]   -> gpurun_out/l1l2_<variant>_<nkr>.csv
vars=$1; n=$2; shift 2
M=gpu__time_duration.sum,smsp__inst_executed.sum,l1tex__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum
for v in $vars; do
  lib=""; [ "$v" != "cur" ] && lib="FSBM_LIB_PATH=build/ab/$v.so"
  env $lib timeout 600 ncu --metrics $M --clock-control none -k regex:coal_dmmag -c 1 --csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-exact --no-configs --nkr $n "$@" \
    > gpurun_out/l1l2_${v}_${n}.csv 2> gpurun_out/l1l2_${v}_${n}.err
  echo "$v $n rc=$?"
done
