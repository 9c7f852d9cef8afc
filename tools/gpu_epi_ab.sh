# A/B of the K3 epilogue: one-shot 32-column TMEM loads (epi0, HEAD) vs double-buffered 16-column loads
# with an early accumulator release (in-tree), and the same with 1 accumulator + 3 A stages (acc1)
mkdir -p gpurun_out
for rep in 1 2; do WLS="cfg2 cfg5 cfg3" STEPS=40 LIBS="paper_2504_19417_b200/libveckm_epi0.so paper_2504_19417_b200/libveckm.so paper_2504_19417_b200/libveckm_acc1.so" bash tools/gpu_ab_lib.sh; done 2>&1 | tee gpurun_out/epi_ab.txt
