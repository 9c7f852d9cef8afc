# launch list + full ncu capture of the hot kernels (one GPU)
mkdir -p gpurun_out
WL=${WL:-cfg2}
KR=${KR:-"k_box_y|k_box_x|k_reduce|k_prep|k_gather_mlp|k_pool"}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${WL}.csv python bench.py --workload $WL --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch_${WL}.log 2>&1; echo "rc ncu-launch $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s ${SKIP:-12} -c ${COUNT:-6} -o gpurun_out/prof_${WL} python bench.py --workload $WL --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${WL}.log 2>&1; echo "rc ncu-full $?"
ls -la gpurun_out
