# A/B of an env switch on the cfg2 bench (kernel breakdown)
for v in 0 1; do
  VKM_TC_PREFETCH=$v timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('prefetch=$v', '%.3e'%d['value'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"
done
