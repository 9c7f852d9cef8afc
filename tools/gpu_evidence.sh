# Round evidence: launch list + full ncu capture of one cfg2 step, bench lines of every config
mkdir -p gpurun_out
make -C paper_2504_19417_b200/csrc -j8 > /dev/null || exit 1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --workload cfg2 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_cfg2.log 2>&1; echo "rc ncu-launch $?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_prep|Radix|Scan|k_scatter|k_runsort|k_longsort|k_reduce|k_box|k_pool|k_gather" -s 20 -c 10 -o gpurun_out/prof_full_cfg2 python bench.py --workload cfg2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_cfg2.log 2>&1; echo "rc ncu-full $?"
[ -n "$ONLY_NCU" ] && exit 0
for wl in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$wl.log 2>&1; echo "rc bench $wl $?"; done
timeout 900 python bench.py > gpurun_out/bench_cfg2.log 2>&1; echo "rc bench cfg2 $?"
ls -la gpurun_out
