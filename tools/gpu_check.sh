set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 300 python tools/tc_check.py cfg1_20k fp32 > gpurun_out/tc_fp32.log 2>&1; echo "rc fp32 $?"
timeout 300 python tools/tc_check.py cfg1_20k f16x3 > gpurun_out/tc_f16.log 2>&1; echo "rc f16 $?"
timeout 300 python tools/tc_check.py cfg1_20k bf16 > gpurun_out/tc_bf16.log 2>&1; echo "rc bf16 $?"
cat gpurun_out/tc_*.log | tail -30
timeout 200 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc smoke $?"; tail -5 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "rc pytest $?"; tail -40 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "rc bench $?"; tail -3 gpurun_out/bench.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "rc ncu1 $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_pool_cplx|k_accumulate|k_gather_mlp|k_features|k_mlp_ffma" -s 5 -c 4 -o gpurun_out/prof_cfg2 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo "rc ncu2 $?"
ls -la gpurun_out
