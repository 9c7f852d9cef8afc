#!/bin/bash
# Build libveckm.so with extra nvcc flags into paper_2504_19417_b200/libveckm_$1.so (A/B with VKM_LIB).
# usage: tools/build_variant.sh NAME "-DVKM_RX_WARPS=1 ..."
set -e
NAME=$1; shift
ROOT=$(cd $(dirname $0)/.. && pwd)
TMP=/tmp/vkm_var_$NAME
rm -rf $TMP && mkdir -p $TMP
mkdir -p $TMP/pkg $TMP/include && cp -r $ROOT/paper_2504_19417_b200/csrc $TMP/pkg/csrc && cp $ROOT/include/*.h $TMP/include/ && rm -f $TMP/pkg/csrc/*.o
sed -i "s|^NVFLAGS := |NVFLAGS := $* |" $TMP/pkg/csrc/Makefile
make -C $TMP/pkg/csrc -j8 OUT=$TMP/libveckm.so > $TMP/build.log 2>&1 || { tail -20 $TMP/build.log; exit 1; }
cp $TMP/libveckm.so $ROOT/paper_2504_19417_b200/libveckm_$NAME.so
echo built paper_2504_19417_b200/libveckm_$NAME.so
