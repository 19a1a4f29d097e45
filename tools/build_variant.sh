#!/bin/bash
# Build an A/B variant of libhefv.so with extra nvcc defines for one source:
#   tools/build_variant.sh NAME SRC.cu -DFOO=1 ...   -> _alt/libhefv_NAME.so
# (select it at run time with HEFV_LIB=_alt/libhefv_NAME.so)
set -e
name=$1; src=$2; shift 2
cd "$(dirname "$0")/.."
mkdir -p _alt/$name
C=paper_1901_10074_b200/csrc
nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC \
  --expt-relaxed-constexpr -Iinclude "$@" -c $C/$src -o _alt/$name/${src%.cu}.o
objs=""
for o in paper_1901_10074_b200/_lib/obj/*.o; do
  b=$(basename $o)
  if [ "$b" == "${src%.cu}.o" ]; then objs="$objs _alt/$name/$b"; else objs="$objs $o"; fi
done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _alt/libhefv_$name.so $objs -lcudart
echo _alt/libhefv_$name.so
