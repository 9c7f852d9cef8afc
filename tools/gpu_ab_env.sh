# A/B of one env switch on the bench (kernel breakdown): VAR=name VALS="0 1" WLS="cfg2 cfg1"
mkdir -p gpurun_out
for wl in ${WLS:-cfg2}; do
for v in ${VALS:-0 1}; do
  env $VAR=$v timeout 300 python bench.py --workload $wl --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl $VAR=$v', '%.3e'%d['value'], round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in (d.get('kernels') or {}).items()})"
done
done
