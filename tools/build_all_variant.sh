#!/bin/bash
# Build an A/B variant of the WHOLE libhefv.so with extra nvcc defines:
#   tools/build_all_variant.sh NAME -DFOO=1 ...   -> _alt/libhefv_NAME.so
# (select it at run time with HEFV_LIB=_alt/libhefv_NAME.so)
set -e
name=$1; shift
cd "$(dirname "$0")/.."
mkdir -p _alt/$name
C=paper_1901_10074_b200/csrc
pids=""
for s in $C/*.cu; do
  b=$(basename ${s%.cu})
  nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -Iinclude "$@" -c $s -o _alt/$name/$b.o &
  pids="$pids $!"
done
for p in $pids; do wait $p; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o _alt/libhefv_$name.so _alt/$name/*.o -lcudart
echo _alt/libhefv_$name.so
