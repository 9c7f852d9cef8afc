# Round evidence on one GPU: smoke, GPU tests, per-config ncu metrics (roofline
# inputs), bench lines of every BASELINE config, the reference arm, two-rank
# shared-GPU lines of the multi-GPU paths, and full ncu captures of the hot
# kernels.  TAG names the files (e.g. v20).
T=${TAG:-cur}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$T.log 2>&1; echo "rc smoke $?"
[ -z "$SKIP_TESTS" ] && { timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$T.log 2>&1; echo "rc pytest $?"; tail -1 gpurun_out/pytest_gpu_$T.log; }
TAG=$T bash tools/gpu_metrics.sh
for wl in cfg1 cfg3 cfg4 cfg5; do timeout 900 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${T}_$wl.jsonl 2>gpurun_out/bench_${T}_$wl.err; echo "rc bench $wl $?"; done
timeout 900 python bench.py > gpurun_out/bench_${T}_cfg2.jsonl 2>gpurun_out/bench_${T}_cfg2.err; echo "rc bench cfg2 $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_${T}_reference_arm.jsonl 2>gpurun_out/bench_${T}_ref.err; echo "rc ref $?"
# N=2 on this one GPU (two ranks sharing cuda:0, gloo plumbing): the timed
# device partition of one slice (config 5 shape) and config 4's 1000 slices
for args in "--workload cfg5 --split spatial" "--workload cfg4"; do
  name=$(echo $args | tr -d ' -' )
  VKM_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline $args > gpurun_out/bench_${T}_n2_$name.jsonl 2>gpurun_out/bench_${T}_n2_$name.err
  echo "rc n2 $name $?"
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather|k_reduce_x|k_box_y" -s 12 -c 3 -o gpurun_out/prof_full_${T}_cfg2 python bench.py --workload cfg2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${T}_cfg2.log 2>&1; echo "rc ncu-full cfg2 $?"
timeout 900 ncu --set full --clock-control none -k regex:"k_gather|k_reduce_x|k_rs_scatter" -s 8 -c 3 -o gpurun_out/prof_full_${T}_cfg5 python bench.py --workload cfg5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full_${T}_cfg5.log 2>&1; echo "rc ncu-full cfg5 $?"
for f in gpurun_out/bench_${T}_*.jsonl; do python -c "import json,sys;d=json.loads(open('$f').readlines()[-1]);print('$f',d.get('config',{}).get('workload','')[:30],'%.3e'%d['value'],'e2e %.3e'%(d.get('e2e') or {}).get('value',0),(d.get('clocks') or {}).get('reasons'))" 2>/dev/null; done
