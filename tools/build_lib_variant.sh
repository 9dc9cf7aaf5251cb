#!/bin/bash
# Build a library variant with extra -D flags (no timeline instrumentation):
#   tools/build_lib_variant.sh NAME -DTB_FUSED_NOQ ...   -> tools/lib_NAME.so
set -e
name=$1; shift
out=/tmp/libvariant_$name; mkdir -p $out
pids=()
for f in abi quantize pack gemv gemv_aux gemm_tc allreduce; do
  rm -f $out/$f.o
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Xcompiler -fPIC,-O3 \
    --expt-relaxed-constexpr "$@" -c paper_2410_16144_b200/csrc/$f.cu -o $out/$f.o &
  pids+=($!)
done
for p in "${pids[@]}"; do wait $p || { echo "compile failed" >&2; exit 1; }; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared $out/*.o -o tools/lib_$name.so -lcudart
echo tools/lib_$name.so
