# bench every BASELINE config on one GPU (no CPU baseline, short)
mkdir -p gpurun_out
for wl in cfg1 cfg2 cfg3 cfg5; do
  timeout 600 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$wl.log 2>&1; echo "rc $wl $?"
  tail -1 gpurun_out/bench_$wl.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'][:40], '%.3e'%d['value'], d['ms_per_step'], {k:round(v['ms'],4) for k,v in (d['kernels'] or {}).items()})" 2>/dev/null
done
timeout 600 python bench.py --workload cfg4 --slices 16 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.log 2>&1; echo "rc cfg4 $?"; tail -1 gpurun_out/bench_cfg4.log | cut -c1-300
