#!/bin/bash
# cfg4 M=8 layer time under library variants / environment switches:
#   tools/build_lib_variant.sh NAME -D...; tools/m8var.sh [VAR=val ...]
run() { echo "== $*"; env "$@" GRAPH=1 timeout 200 python tools/ncu_stack.py cfg4 i2s 8 16 2>&1 | tail -1; }
run A=default
run TB_M8_GLUE_FIN=0
run TB_M8_PIPELINED=0
for v in "$@"; do run $v; done
