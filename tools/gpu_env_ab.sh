# A/B of env settings on the bench: ENVS="A=1 B=2;A=3" (';' separates variants), WLS workloads
mkdir -p gpurun_out
make -C paper_2504_19417_b200/csrc -j8 > /dev/null || exit 1
if [ -n "$TESTS" ]; then timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "rc pytest $?"; tail -3 gpurun_out/pytest_gpu.log; fi
bl() { timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3e'%d['value'], round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in (d['kernels'] or {}).items()})"; }
IFS=';' read -ra VARS <<< "${ENVS:-X=0}"
for wl in ${WLS:-cfg2}; do
  for v in "${VARS[@]}"; do echo "== $wl [$v]"; env $v bash -c "$(declare -f bl); bl --workload $wl"; done
done
