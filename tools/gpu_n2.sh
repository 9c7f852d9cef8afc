# Two ranks sharing the one GPU (gloo plumbing): the multi-GPU bench paths
T=${TAG:-cur}
mkdir -p gpurun_out
for args in "--workload cfg5 --split spatial" "--workload cfg4" "--workload cfg2"; do
  name=$(echo $args | tr -d ' -' )
  VKM_BENCH_SHARED_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --no-cpu-baseline $args > gpurun_out/bench_${T}_n2_$name.jsonl 2>gpurun_out/bench_${T}_n2_$name.err
  echo "rc n2 $name $?"; tail -1 gpurun_out/bench_${T}_n2_$name.jsonl | cut -c1-400
done
