# quick GPU loop: mode check + full GPU test suite + short bench
mkdir -p gpurun_out
for m in fp32 f16x3 bf16; do timeout 300 python tools/tc_check.py cfg1_20k $m 2>&1 | tail -2; done
timeout 200 python __graft_entry__.py smoke 2>&1 | tail -2
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "rc pytest $?"; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "rc bench $?"; tail -2 gpurun_out/bench.log
