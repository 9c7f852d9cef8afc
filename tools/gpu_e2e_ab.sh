# e2e A/B of the host packing switch: VALS="0 1" WLS="cfg2 cfg4"
mkdir -p gpurun_out
for wl in ${WLS:-cfg2}; do
for v in ${VALS:-0 1}; do
  VKM_HOST_PACK=$v timeout 600 python bench.py --workload $wl --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$wl pack=$v', 'value %.3e'%d['value'], 'e2e %.3e'%e['value'], 'single %.3e'%e['single_slice']['value'], 'h2d', e['h2d_bytes_per_step'])"
done
done
