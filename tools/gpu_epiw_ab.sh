# A/B of the K3 epilogue warp count: 4 (libveckm_epi4.so) vs 8 (in-tree)
mkdir -p gpurun_out
for rep in 1 2; do WLS="cfg2 cfg5 cfg3 cfg1" STEPS=40 LIBS="paper_2504_19417_b200/libveckm_epi4.so paper_2504_19417_b200/libveckm.so" bash tools/gpu_ab_lib.sh; done 2>&1 | tee gpurun_out/epiw_ab.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/pytest_epiw.log 2>&1; echo rc pytest $?; tail -1 gpurun_out/pytest_epiw.log
