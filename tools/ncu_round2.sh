#!/bin/bash
# Round-2 ncu evidence (one gpurun call; each ncu preceded by its plain run).
set -u
O=gpurun_out/ncu2; mkdir -p $O
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,dram__bytes_read.sum.per_second,dram__throughput.avg.pct_of_peak_sustained_elapsed,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__inst_executed.sum
for w in "cfg4 8" "cfg1 48" "cfg2tl2 8" "cfg2i2s 8" "cfg4m8 4"; do
  set -- $w
  python tools/ncu_graph.py $1 $2 > $O/plain_$1.log 2>&1 && \
  ncu --graph-profiling graph --nvtx --nvtx-include "prof/" --metrics $M --clock-control none \
      --csv --log-file $O/graph_$1.csv python tools/ncu_graph.py $1 $2 > $O/ncu_$1.log 2>&1
  echo "$1 rc=$?"
done
# full sets of the top kernels (single launches inside the graph replay)
python tools/ncu_graph.py cfg4 4 > $O/plain_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on --graph-profiling node --nvtx --nvtx-include "prof/" \
    -k regex:tgemv_kernel -c 2 -o $O/cfg4_step_full python tools/ncu_graph.py cfg4 4 > $O/ncu_full.log 2>&1
echo "full cfg4 rc=$?"
python tools/ncu_graph.py cfg2tl2 4 > $O/plain_fulltl2.log 2>&1 && \
ncu --set full --clock-control none --import-source on --graph-profiling node --nvtx --nvtx-include "prof/" \
    -k regex:tgemv_kernel -c 2 -o $O/tl2_step_full python tools/ncu_graph.py cfg2tl2 4 > $O/ncu_fulltl2.log 2>&1
echo "full tl2 rc=$?"
