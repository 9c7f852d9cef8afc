# e2e A/B of the mixed packed/raw transfer (VKM_PACK_RAW_EVERY), 3 runs each, alternating
mkdir -p gpurun_out
for rep in 1 2 3; do
for m in 0 2 3 4; do
  VKM_PACK_RAW_EVERY=$m timeout 300 python bench.py --workload ${WL:-cfg2} --steps 40 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${WL:-cfg2} raw_every=$m', 'e2e %.3e'%d['e2e']['value'], 'single %.3e'%d['e2e']['single_slice']['value'])"
done; done
