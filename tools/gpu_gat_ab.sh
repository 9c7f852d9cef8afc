# A/B of the K3 block gather: HEAD's per-pair gather (libveckm_red2.so), all
# rows loaded up front (libveckm_gat.so, VKM_K3_LDSPLIT=0), second half loaded
# mid-tile (in-tree build)
mkdir -p gpurun_out
for rep in 1 2; do
  WLS="cfg2 cfg5 cfg3 cfg1" STEPS=40 LIBS="paper_2504_19417_b200/libveckm_red2.so paper_2504_19417_b200/libveckm_gat.so paper_2504_19417_b200/libveckm.so" bash tools/gpu_ab_lib.sh
done 2>&1 | tee gpurun_out/gat_ab2.txt
