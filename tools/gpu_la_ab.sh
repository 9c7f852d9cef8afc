# A/B of the K3 producers' pooled-row load schedule: per half (split) vs pair u+L loaded at pair u (la2..la6)
mkdir -p gpurun_out
L="paper_2504_19417_b200/libveckm_split.so"; for v in la2 la3 la4 la6; do L="$L paper_2504_19417_b200/libveckm_$v.so"; done
for rep in 1 2; do WLS="cfg2 cfg5 cfg3" STEPS=40 LIBS="$L" bash tools/gpu_ab_lib.sh; done 2>&1 | tee gpurun_out/la_ab.txt
