# e2e (pinned host batch) and drop-in predict under two host-pool granularities, alternating
for r in 1 2 3; do
  for g in 32768 8192; do
    VKM_PACK_GRAIN=$g timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('grain $g', 'value %.3e'%d['value'], 'e2e %.3e'%d['e2e']['value'])"
  done
done
for g in 32768 8192; do VKM_PACK_GRAIN=$g python tools/prof_predict.py 2>&1 | head -1 | sed "s/^/grain $g /"; done
