# A/B: long runs sorted inside k_runsort (in-tree) vs the separate k_longsort launch (libveckm_lsk.so)
mkdir -p gpurun_out
for rep in 1 2; do WLS="cfg1 cfg2 cfg3 cfg4" STEPS=40 LIBS="paper_2504_19417_b200/libveckm_lsk.so paper_2504_19417_b200/libveckm.so" bash tools/gpu_ab_lib.sh; done 2>&1 | tee gpurun_out/lsk_ab.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_lsk.log 2>&1; echo rc pytest $?; tail -1 gpurun_out/pytest_lsk.log
