# ncu of coal_dmma with the dense vs the line-aligned compaction (C2)
M=gpu__time_duration.sum,smsp__inst_executed.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__sass_thread_inst_executed_op_dmma_pred_on.sum,smsp__inst_executed_pipe_fp64.sum,dram__bytes_read.sum
for v in dense lined; do
  env=""; [ $v = dense ] && env="FSBM_DENSE_COMPACTION=1"
  env $env timeout 600 ncu --metrics $M --clock-control none -k regex:coal_dmma_kernel -c 1 --csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-exact --no-configs > gpurun_out/nl_$v.csv 2>/dev/null
done
