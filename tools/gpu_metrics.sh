# Per-config ncu metrics of the bench's kernels (one GPU): duration, DRAM bytes,
# warp instructions, pipe utilisation (FMA / ALU / XU / tensor), issue and warp
# activity.  Parsed by tools/ncu_roofline.py into profiles/ncu_{traffic,instr,pipes}.json.
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum
M=$M,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__inst_executed_pipe_tc.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_xu.sum
M=$M,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active
M=$M,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active
M=$M,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active
M=$M,sm__cycles_elapsed.avg.per_second
for wl in ${WLS:-cfg1 cfg2 cfg3 cfg4 cfg5}; do
  timeout ${NCU_TIMEOUT:-600} ncu --metrics $M --clock-control none -k regex:"^k_|Device|Onesweep" --csv --page raw \
    --log-file gpurun_out/metrics_${TAG:-cur}_$wl.csv python bench.py --workload $wl --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline > gpurun_out/metrics_${TAG:-cur}_$wl.log 2>&1
  echo "rc metrics $wl $?"
done
