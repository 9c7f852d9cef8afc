L=paper_2504_19417_b200
run() { timeout 300 python bench.py --workload $1 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', '%.3e'%d['value'], {k:round(v['ms'],4) for k,v in d['kernels'].items()})"; }
for wl in cfg2 cfg5; do
  VKM_LIB=$PWD/$L/libveckm_probedx.so run $wl base
  for seg in 0 64 32; do VKM_RX_SEG=$seg VKM_RX_DXP=3 VKM_LIB=$PWD/$L/libveckm_probedx.so run $wl "dx3 seg=$seg"; done
  VKM_LIB=$PWD/$L/libveckm_probe.so run $wl "y3tap (dx10)"
done
