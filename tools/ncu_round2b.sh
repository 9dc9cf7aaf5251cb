#!/bin/bash
# Round-2 (second pass) ncu evidence after the M=8 table mode and TL2 v-tiles.
set -u
O=gpurun_out/ncu2b; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum
python tools/ncu_graph.py cfg4m8 4 > $O/plain_m8.log 2>&1 && \
ncu --graph-profiling graph --nvtx --nvtx-include "prof/" --metrics $M --clock-control none \
    --csv --log-file $O/graph_cfg4m8.csv python tools/ncu_graph.py cfg4m8 4 > $O/ncu_m8g.log 2>&1
echo "m8 graph rc=$?"
python tools/ncu_graph.py cfg4m8 2 > $O/plain_m8f.log 2>&1 && \
ncu --set full --clock-control none --import-source on --graph-profiling node --nvtx --nvtx-include "prof/" \
    -k regex:tgemv_kernel -c 1 -o $O/m8_table_full python tools/ncu_graph.py cfg4m8 2 > $O/ncu_m8f.log 2>&1
echo "m8 full rc=$?"
python tools/ncu_graph.py cfg2tl2 4 > $O/plain_tl2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --graph-profiling node --nvtx --nvtx-include "prof/" \
    -k regex:tgemv_kernel -c 1 -o $O/tl2v_full python tools/ncu_graph.py cfg2tl2 4 > $O/ncu_tl2.log 2>&1
echo "tl2 full rc=$?"
