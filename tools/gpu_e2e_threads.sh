# e2e (pinned host batch, cfg2) vs host pool size, alternating
for r in 1 2; do
  for t in 16 8 12 6; do
    VKM_HOST_THREADS=$t timeout 300 python bench.py --workload cfg2 --steps 20 --warmup 3 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads $t', 'e2e %.3e'%d['e2e']['value'])"
  done
done
