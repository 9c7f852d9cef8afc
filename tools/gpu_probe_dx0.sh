L=paper_2504_19417_b200
for wl in cfg2 cfg5 cfg3; do
  for seg in 0 32 64 128; do
    VKM_RX_SEG=$seg VKM_RX_DX0=1 VKM_LIB=$PWD/$L/libveckm_dx0.so timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl dx0 seg=$seg', {k:round(v['ms'],4) for k,v in (d.get('kernels') or {}).items()})"
  done
  VKM_LIB=$PWD/$L/libveckm_dx0.so timeout 300 python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$wl base', {k:round(v['ms'],4) for k,v in (d.get('kernels') or {}).items()})"
done
VKM_RX_DX0=1 VKM_LIB=$PWD/$L/libveckm_dx0.so timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_reduce_x|k_run_starts" -c 2 python bench.py --workload cfg5 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_reduce|k_run|duration|warps|issue"
VKM_RX_DX0=1 VKM_LIB=$PWD/$L/libveckm_dx0.so timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:"k_reduce_x" -c 1 python bench.py --workload cfg2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>&1 | grep -E "k_reduce|duration|warps|issue"
