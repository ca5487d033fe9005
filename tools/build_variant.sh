#!/bin/bash
# Build a libdffm.so variant with extra nvcc defines (A/B of compile-time knobs):
#   tools/build_variant.sh NAME -DDFFM_RSW_NMW=4 ...   ->  build_var/NAME/libdffm.so
# Select it at run time with DFFM_LIB_PATH=build_var/NAME/libdffm.so.
set -e
NAME=$1; shift
OUT=build_var/$NAME
mkdir -p $OUT
SRC=${SRC:-paper_2407_10115_b200/csrc}
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $*"
pids=()
for f in $SRC/*.cu; do
  b=$(basename $f .cu)
  nvcc $FLAGS -c $f -o $OUT/$b.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -o $OUT/libdffm.so $OUT/*.o
echo built $OUT/libdffm.so
