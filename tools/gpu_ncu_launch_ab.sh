# per-kernel launch times (ncu, serialised) for several builds: LIBS="a.so b.so" KR=regex
mkdir -p gpurun_out
for lib in ${LIBS}; do
  nm=$(basename $lib .so)
  VKM_LIB=$PWD/$lib timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KR:-.}" --csv --log-file gpurun_out/la_$nm.csv python bench.py --workload ${WL:-cfg2} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
  echo "== $nm"; python tools/ncu_summary.py gpurun_out/la_$nm.csv 2>/dev/null | grep -v FillFun
done
