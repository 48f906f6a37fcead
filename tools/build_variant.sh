#!/bin/bash
# build an A/B variant of libboys: tools/build_variant.sh <name> [-DMACRO=..]...  -> ab_libs/libboys_<name>.so
# (only ragged.cu / dense.cu are recompiled with the macros; the other objects come from paper_2504_07637_b200/build)
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p ab_libs /tmp/abobj_$name
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC"
for u in ${UNITS:-ragged}; do
  nvcc $FL "$@" -c -o /tmp/abobj_$name/$u.o paper_2504_07637_b200/csrc/$u.cu &
done
wait
objs=""
for u in dense ragged split table shard hermite abi; do
  if [ -f /tmp/abobj_$name/$u.o ]; then objs="$objs /tmp/abobj_$name/$u.o"; else objs="$objs paper_2504_07637_b200/build/$u.o"; fi
done
nvcc $FL -shared -o ab_libs/libboys_$name.so $objs
echo built ab_libs/libboys_$name.so
