#!/bin/bash
# Build a timeline-instrumented variant of the library with extra -D flags:
#   tools/build_variant.sh NAME -DTB_MT1_RING=2 ...   -> tools/lib_NAME.so
set -e
name=$1; shift
out=/tmp/variant_$name; mkdir -p $out
pids=()
for f in abi quantize pack gemv gemv_aux gemm_tc allreduce; do
  rm -f $out/$f.o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC -DTB_TIMELINE "$@" \
    -c paper_2410_16144_b200/csrc/$f.cu -o $out/$f.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "compile failed" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared $out/*.o -o tools/lib_$name.so
echo tools/lib_$name.so
