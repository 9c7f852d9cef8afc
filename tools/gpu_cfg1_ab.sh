# Small-slice (config 1) k_reduce_x A/B: segment width and the one-channel-per-lane variant
for v in "VKM_RX_SEG=0" "VKM_RX_SEG=64" "VKM_RX_SEG=128" "VKM_RX=1" "VKM_RX_SEG=0"; do
  env $v timeout 300 python bench.py --workload cfg1 --steps 50 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 $v', '%.3e'%d['value'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"
done
