# iteration loop: GPU tests (default path), split-path parity subset, A/B bench of pooling paths and segment widths
mkdir -p gpurun_out
make -C paper_2504_19417_b200/csrc -j8 > /dev/null || exit 1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "rc pytest $?"; tail -15 gpurun_out/pytest_gpu.log
bl() { timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu-baseline --no-e2e "$@" 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3e'%d['value'], round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in d['kernels'].items()})"; }
for wl in ${WLS:-cfg2}; do
  echo "== $wl split"; VKM_POOL=split bl --workload $wl
  echo "== $wl fused"; bl --workload $wl
  for sg in ${SEGS:-}; do echo "== $wl fused seg $sg"; VKM_RX_SEG=$sg bl --workload $wl; done
done
