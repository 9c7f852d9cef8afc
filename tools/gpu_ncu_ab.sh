# full ncu of one kernel per build/env variant: KR=regex, VARIANTS="name:ENV=..:lib ..."
mkdir -p gpurun_out
for v in ${VARIANTS}; do
  name=${v%%:*}; rest=${v#*:}; envs=${rest%%:*}; lib=${rest#*:}
  env $envs VKM_LIB=$PWD/$lib timeout 300 ncu --set full --clock-control none --import-source on -k regex:"$KR" -s ${SKIP:-6} -c 1 -o gpurun_out/ab_$name python bench.py --workload ${WL:-cfg2} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_$name.log 2>&1; echo "rc $name $?"
done
