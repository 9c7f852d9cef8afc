# ncu full of K3 at cfg2 for HEAD's per-pair gather (red2) and the in-tree block gather
mkdir -p gpurun_out
for v in red2 cur; do
  lib=$PWD/paper_2504_19417_b200/libveckm_$v.so; [ $v = cur ] && lib=$PWD/paper_2504_19417_b200/libveckm.so
  VKM_LIB=$lib timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_gather" -s 4 -c 1 -o gpurun_out/k3_$v python bench.py --workload cfg2 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/k3_$v.log 2>&1; echo "rc $v $?"
done
