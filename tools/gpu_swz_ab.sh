# A/B of the pooled-grid chunk swizzle (in-tree, VKM_Q_SWZ=1) against the linear layout (libveckm_noswz.so)
mkdir -p gpurun_out
for rep in 1 2; do WLS="cfg2 cfg5 cfg3 cfg1" STEPS=40 LIBS="paper_2504_19417_b200/libveckm_noswz.so paper_2504_19417_b200/libveckm.so" bash tools/gpu_ab_lib.sh; done 2>&1 | tee gpurun_out/swz_ab.txt
VKM_PARITY_OUT=$PWD/gpurun_out/parity_atsize_v29_mufu.jsonl timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_v29.log 2>&1; echo rc pytest $?; tail -1 gpurun_out/pytest_gpu_v29.log
