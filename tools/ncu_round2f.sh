#!/bin/bash
# Final round-2 ncu evidence: the pipelined cfg4 M=8 layers (graph-level bytes
# of a 4-layer chain; one full capture of the records-table GEMV).
set -u
O=gpurun_out/ncu2f; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed.sum
python tools/ncu_graph.py cfg4m8 4 > $O/plain_m8.log 2>&1 && \
timeout 600 ncu --graph-profiling graph --nvtx --nvtx-include "prof/" --metrics $M --clock-control none \
    --csv --log-file $O/graph_cfg4m8.csv python tools/ncu_graph.py cfg4m8 4 > $O/ncu_m8g.log 2>&1
echo "m8 graph rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on --graph-profiling node --nvtx --nvtx-include "prof/" \
    -k regex:tgemv_kernel -s 1 -c 1 -o $O/m8_piped_full python tools/ncu_graph.py cfg4m8 3 > $O/ncu_m8f.log 2>&1
echo "m8 full rc=$?"
ncu -i $O/m8_piped_full.ncu-rep --page details > $O/m8_piped_full.txt 2>/dev/null
