# K1 iteration check on one GPU: GPU tests, cfg2/cfg5 bench lines, launch lists
mkdir -p gpurun_out
T=${TAG:-k1}
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 ${PYK:+-k "$PYK"} > gpurun_out/pytest_$T.log 2>&1; echo "rc pytest $?"; tail -4 gpurun_out/pytest_$T.log
for wl in ${WLS:-cfg2 cfg5}; do
  timeout 600 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_${T}_$wl.log 2>&1; echo "rc bench $wl $?"
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${T}_$wl.csv python bench.py --workload $wl --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1; echo "rc ncu $wl $?"
done
