# full round check on one GPU: smoke, GPU tests, default bench (with CPU baseline), reference arm, launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
lscpu | grep -E "Model name|^CPU\(s\)" ; nproc
timeout 200 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "rc smoke $?"; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "rc pytest $?"; tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "rc bench $?"; tail -2 gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "rc ref $?"; tail -2 gpurun_out/bench_ref.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg2.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "rc ncu-launch $?"
