# A/B of the MUFU argument reduction (VKM_MUFU_RED 2/1/0 builds): bench of
# configs 2, 5, 3 (alternating builds, twice) and at-size + golden parity.
mkdir -p gpurun_out
for rep in 1 2; do
  WLS="cfg2 cfg5 cfg3" STEPS=40 LIBS="paper_2504_19417_b200/libveckm_red2.so paper_2504_19417_b200/libveckm_red0.so paper_2504_19417_b200/libveckm_red1.so" bash tools/gpu_ab_lib.sh
done 2>&1 | tee gpurun_out/red_ab.txt
for v in red2 red0 red1; do
  VKM_LIB=$PWD/paper_2504_19417_b200/libveckm_$v.so VKM_PARITY_OUT=$PWD/gpurun_out/parity_$v.jsonl timeout 900 \
    python -m pytest tests/test_gpu_atsize.py tests/test_gpu_parity.py -m gpu -q -x > gpurun_out/pytest_$v.log 2>&1
  echo "rc $v $?"; tail -1 gpurun_out/pytest_$v.log
done
