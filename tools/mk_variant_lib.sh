#!/bin/bash
# Build ab/lib_$1.so: the in-tree objects (build/native) with the units named
# in $UNITS (default: wilson) recompiled with the extra nvcc flags "$2".
# Usage: tools/mk_variant_lib.sh ld1 "-DMGT_PIPE_LD=1"; then on the GPU box
#   MGT_LIB_PATH=ab/lib_ld1.so python tools/sweep.py ...
set -e
NAME=$1; EXTRA=$2; UNITS=${UNITS:-wilson}
mkdir -p ab/obj_$NAME
OBJS=""
for o in build/native/*.o; do
  b=$(basename $o .o)
  if [[ " $UNITS " == *" $b "* ]]; then
    /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 \
      -Xptxas -v --expt-relaxed-constexpr -Iinclude $EXTRA -c paper_1909_12234_b200/csrc/$b.cu -o ab/obj_$NAME/$b.o \
      > ab/obj_$NAME/$b.log 2>&1
    OBJS="$OBJS ab/obj_$NAME/$b.o"
  else
    OBJS="$OBJS $o"
  fi
done
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ab/lib_$NAME.so $OBJS -lcudart_static -lrt -ldl -lpthread
rm -rf ab/obj_$NAME/*.o
echo built ab/lib_$NAME.so
