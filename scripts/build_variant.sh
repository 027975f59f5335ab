#!/bin/bash
# Build a variant of libspgb200.so with extra -D flags (dev tool):
#   scripts/build_variant.sh NAME "-DSPG_NB_SHIFT=0 ..."  -> var/NAME/libspgb200.so
set -e -o pipefail
NAME=$1; shift
FLAGS="$*"
OUT=var/$NAME
mkdir -p $OUT/obj
for f in paper_2603_21444_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  nvcc -O3 -lineinfo -std=c++17 -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -Iinclude \
       -Ipaper_2603_21444_b200/csrc --expt-relaxed-constexpr $FLAGS -c $f -o $OUT/obj/$b.o &
done
for j in $(jobs -p); do wait $j || exit 1; done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libspgb200.so $OUT/obj/*.o -cudart static
rm -rf $OUT/obj
echo built $OUT/libspgb200.so
