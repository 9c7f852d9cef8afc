# A/B of two builds on the bench: LIBS="paper_2504_19417_b200/libveckm_head.so paper_2504_19417_b200/libveckm.so"
mkdir -p gpurun_out
for wl in ${WLS:-cfg2}; do
for lib in ${LIBS}; do
  VKM_LIB=$PWD/$lib timeout 300 python bench.py --workload $wl --steps ${STEPS:-50} --warmup 5 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl $(basename $lib) ${EXTRA}', '%.3e'%d['value'], round(d['ms_per_step'],4), {k:round(v['ms'],4) for k,v in (d.get('kernels') or {}).items()})"
done
done
