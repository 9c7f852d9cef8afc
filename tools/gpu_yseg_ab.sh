# y-pass segment count A/B (VKM_YSEGS; 0 = automatic)
for wl in cfg2 cfg5 cfg3; do
  for s in 0 6 8 12 16 0; do
    VKM_YSEGS=$s timeout 300 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl segs=$s', '%.3e'%d['value'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"
  done
done
