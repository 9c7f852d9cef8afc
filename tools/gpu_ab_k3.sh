# K3 A/B: library variants and the L2-prefetch switch on cfg2
mkdir -p gpurun_out
L=paper_2504_19417_b200
LIBS="$L/libveckm_mufu.so $L/libveckm_qd2.so $L/libveckm_phb4.so $L/libveckm_phb1.so $L/libveckm_mufu.so" bash tools/gpu_ab_lib.sh
VKM_TC_PREFETCH=0 LIBS="$L/libveckm_mufu.so" EXTRA=noprefetch bash tools/gpu_ab_lib.sh
